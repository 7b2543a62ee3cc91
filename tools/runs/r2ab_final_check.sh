# round 2, call AB (4 GPUs): final push launcher -- fast tier, multi-GPU parity, smoke
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ab_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py tests/test_readme_example.py tests/test_heap_cpu.py -q -m "gpu and not slow or not gpu" -k "not gloo" > gpurun_out/r2ab_pytest.log 2>&1
echo pytest_rc=$?
timeout 2000 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/r2ab_pytest_multi.log 2>&1
echo multi_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ab_smoke.log 2>&1
echo smoke_rc=$?
tail -1 gpurun_out/r2ab_pytest.log; tail -1 gpurun_out/r2ab_pytest_multi.log; tail -1 gpurun_out/r2ab_smoke.log
