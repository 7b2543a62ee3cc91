# round 2, call H (1 GPU): per-segment checksum flush in K1/K2 -- parity, in-situ decomposition, N=1 bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py -q -m "gpu and not slow" > gpurun_out/r2h_pytest.log 2>&1
echo pytest_rc=$?
timeout 900 python tools/pack_insitu.py --model qwen2.5-7b --variants 0 --out gpurun_out/r2h_pack_insitu.jsonl > gpurun_out/r2h_pack_insitu.log 2>&1
echo insitu_rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2h_bench.log 2>&1
echo bench_rc=$?
tail -3 gpurun_out/r2h_pytest.log
python - <<'PY'
import json
for l in open("gpurun_out/r2h_pack_insitu.jsonl"):
    d = json.loads(l); pb = d.pop("per_bucket", None); print(d)
    if pb and d.get("mode") == "gap":
        print("   slow buckets:", [(b["bucket"], b["us"]) for b in pb if b["segments"] <= 5])
PY
grep '^{' gpurun_out/r2h_bench.log | tail -1 | cut -c1-300
grep -o '"roofline": {[^}]*}' gpurun_out/r2h_bench.log
