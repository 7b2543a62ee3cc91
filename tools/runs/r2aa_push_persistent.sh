# round 2, call AA (4 GPUs): persistent grid-stride push (PLEX_PUSH_PERSISTENT=1) vs one CTA per item --
# parity of the sync tests with the variant, then a same-box A/B of the push probe
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aa_build.log 2>&1
PLEX_PUSH_PERSISTENT=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -k "sync or push or replica or multiplex or group or gather" > gpurun_out/r2aa_pytest_persist.log 2>&1
echo pytest_rc=$?
PLEX_PUSH_PERSISTENT=1 timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "collective" > gpurun_out/r2aa_pytest_multi_persist.log 2>&1
echo multi_rc=$?
for pass in 1 2; do
  for v in 0 1; do
    for only in all row; do
      PLEX_PUSH_PERSISTENT=$v timeout 600 python tools/push_probe.py --gpus 4 --model qwen2.5-7b --tp 2 --only $only --out gpurun_out/r2aa_probe_v$v.jsonl > /dev/null 2>&1
    done
    PLEX_PUSH_PERSISTENT=$v timeout 600 python tools/push_probe.py --gpus 4 --model qwen2.5-32b --tp 4 --only all --out gpurun_out/r2aa_probe_v$v.jsonl > /dev/null 2>&1
    PLEX_PUSH_PERSISTENT=$v timeout 600 python tools/push_probe.py --gpus 2 --model qwen2.5-7b --tp 2 --only all --out gpurun_out/r2aa_probe_v$v.jsonl > /dev/null 2>&1
  done
done
tail -1 gpurun_out/r2aa_pytest_persist.log gpurun_out/r2aa_pytest_multi_persist.log
for v in 0 1; do echo v=$v; python -c "
import json,sys
for l in open('gpurun_out/r2aa_probe_v$v.jsonl'):
    d=json.loads(l); print(d['model'], d['n_gpus'], d['only'], d['push_ms_max_rank'], d['nvlink_gbs'], d['frac_of_bound'])
"; done
