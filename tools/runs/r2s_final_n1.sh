# round 2, call S (1 GPU): 8-piece swap default -- fast parity tier, full-size 7B swap, final N=1 bench line
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py tests/test_readme_example.py -q -m "gpu and not slow" > gpurun_out/r2s_pytest.log 2>&1
echo pytest_rc=$?
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k "swap" > gpurun_out/r2s_pytest_swap7b.log 2>&1
echo swap7b_rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2s_bench.log 2>&1
echo bench_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1
echo smoke_rc=$?
tail -1 gpurun_out/r2s_pytest.log gpurun_out/r2s_pytest_swap7b.log
grep '^{' gpurun_out/r2s_bench.log | tail -1 | cut -c1-400
