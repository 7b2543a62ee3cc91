# round 2, call I (4 GPUs): multi-GPU parity + N=2 / N=4 bench with the final kernels
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2i_topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_multi.py -v -m gpu --durations=0 > gpurun_out/r2i_pytest_multi.log 2>&1
echo pytest_rc=$?
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2i_bench_n2.log 2>&1
echo bench2_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2i_bench_n4.log 2>&1
echo bench4_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --steps 5 --warmup 3 --impl reference > gpurun_out/r2i_bench_n4_ref.log 2>&1
echo ref4_rc=$?
tail -3 gpurun_out/r2i_pytest_multi.log
for n in 2 4; do grep '^{' gpurun_out/r2i_bench_n$n.log | tail -1 | cut -c1-400; done
grep '^{' gpurun_out/r2i_bench_n4_ref.log | tail -1 | cut -c1-300
