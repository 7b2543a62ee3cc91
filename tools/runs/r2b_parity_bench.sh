# round 2, call B: GPU parity (not slow) + bench contract + short N=1 bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py -q -m "gpu and not slow" > gpurun_out/r2b_pytest.log 2>&1
echo pytest_rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2b_bench.log 2>&1
echo bench_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
echo smoke_rc=$?
tail -c 4000 gpurun_out/r2b_bench.log
tail -15 gpurun_out/r2b_pytest.log
