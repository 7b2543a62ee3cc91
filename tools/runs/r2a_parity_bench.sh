# round 2, call A: build, GPU parity (not slow), short N=1 bench
set -x
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/r2a_pytest.log 2>&1
echo pytest_rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2a_bench.log 2>&1
echo bench_rc=$?
tail -c 3000 gpurun_out/r2a_bench.log
tail -5 gpurun_out/r2a_pytest.log
