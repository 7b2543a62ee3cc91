# round 2, call G (1 GPU): staging-offset sweep of the single-tensor buckets (pack_insitu --shift-sweep)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1
timeout 900 python tools/pack_insitu.py --model qwen2.5-7b --shift-sweep --out gpurun_out/r2g_shift.jsonl > gpurun_out/r2g_shift.log 2>&1
echo rc=$?
cat gpurun_out/r2g_shift.jsonl
tail -5 gpurun_out/r2g_shift.log
