# round 2, call F (1 GPU): pack/unpack in-situ decomposition (fixed: no pointer upload in the timed launches)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1
timeout 900 python tools/pack_insitu.py --model qwen2.5-7b --out gpurun_out/r2f_pack_insitu.jsonl > gpurun_out/r2f_pack_insitu.log 2>&1
echo insitu_rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/r2f_pack_insitu.jsonl"):
    d = json.loads(l); d.pop("per_bucket", None); print(d)
PY
