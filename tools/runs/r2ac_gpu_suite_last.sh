# round 2, call AC (1 GPU): the driver's GPU tier exactly as it runs it (pytest -m gpu) + smoke
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ac_build.log 2>&1
timeout 3300 python -m pytest tests/ -x -q -m gpu --durations=40 > gpurun_out/r2ac_pytest_gpu_all.log 2>&1
echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ac_smoke.log 2>&1
echo smoke_rc=$?
tail -50 gpurun_out/r2ac_pytest_gpu_all.log
