# round 2, call L (1 GPU): configs[4] multiplex trace (D1: 5 rounds, 19 switches) and the NEXT-4 HRRS
# scenario, both through the group executor
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
timeout 1200 python tools/scenarios.py --scenario multiplex --gpus 1 --out gpurun_out/r2l_scen.jsonl > gpurun_out/r2l_multiplex.log 2>&1
echo multiplex_rc=$?
timeout 1200 python tools/scenarios.py --scenario hrrs --gpus 1 --out gpurun_out/r2l_scen.jsonl > gpurun_out/r2l_hrrs.log 2>&1
echo hrrs_rc=$?
cat gpurun_out/r2l_scen.jsonl
tail -3 gpurun_out/r2l_multiplex.log gpurun_out/r2l_hrrs.log
