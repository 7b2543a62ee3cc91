# round 2, call M (4 GPUs): a same-box scaling curve N=1/2/4 of the bench (as the driver's SCALE run does),
# then the configs[4] multiplex trace through the group executor at N=4 (D1: 5 rounds, 19 switches)
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2m_topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_bench_n1.log 2>&1
echo bench1_rc=$?
timeout 900 $TR --nproc-per-node 2 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2m_bench_n2.log 2>&1
echo bench2_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29532 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2m_bench_n4.log 2>&1
echo bench4_rc=$?
timeout 1500 $TR --nproc-per-node 4 --master-port 29533 tools/scenarios.py --scenario multiplex --gpus 4 --out gpurun_out/r2m_scen.jsonl > gpurun_out/r2m_multiplex4.log 2>&1
echo mplex4_rc=$?
for n in 1 2 4; do grep '^{' gpurun_out/r2m_bench_n$n.log | tail -1 | cut -c1-300; done
cat gpurun_out/r2m_scen.jsonl
