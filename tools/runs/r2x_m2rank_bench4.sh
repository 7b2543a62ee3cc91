# round 2, call X (4 GPUs): host-bandwidth probe of the box, M2 per-GPU workload at k = 4, N=4 and N=2 bench
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2x_topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29571 tools/scenarios.py --scenario m2rank --gpus 4 --steps 6 --warmup 2 --out gpurun_out/r2x_scen.jsonl > gpurun_out/r2x_m2rank4.log 2>&1
echo k4_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29572 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2x_bench_n4.log 2>&1
echo bench4_rc=$?
timeout 900 $TR --nproc-per-node 2 --master-port 29573 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2x_bench_n2.log 2>&1
echo bench2_rc=$?
cat gpurun_out/r2x_scen.jsonl
for n in 2 4; do grep '^{' gpurun_out/r2x_bench_n$n.log | tail -1 | cut -c1-250; done
