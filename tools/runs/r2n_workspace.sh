# round 2, call N (4 GPUs): caller-owned workspace refactor -- fast GPU parity tier, multi-GPU parity
# (carry flags exported over IPC from the workspace), short N=1 / N=4 bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py tests/test_readme_example.py -q -m "gpu and not slow" > gpurun_out/r2n_pytest.log 2>&1
echo pytest_rc=$?
timeout 2000 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/r2n_pytest_multi.log 2>&1
echo multi_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1
echo smoke_rc=$?
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29541 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r2n_bench_n4.log 2>&1
echo bench4_rc=$?
tail -3 gpurun_out/r2n_pytest.log gpurun_out/r2n_pytest_multi.log
grep '^{' gpurun_out/r2n_bench_n4.log | tail -1 | cut -c1-250
