# round 2, call C: full-size config parity (slow tier) on one B200
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
nproc > gpurun_out/r2c_nproc.txt
timeout 3000 python -m pytest tests/test_gpu_fullsize_configs.py -v -m gpu --durations=0 > gpurun_out/r2c_pytest_fullsize.log 2>&1
echo pytest_rc=$?
tail -30 gpurun_out/r2c_pytest_fullsize.log
