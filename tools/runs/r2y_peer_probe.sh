# round 2, call Y (4 GPUs): NVLink copy-engine denominators (pair / bidirectional / all-to-all) next to the
# fused push on the same box
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1
timeout 600 python tools/peer_probe.py --gpus 4 --gb 4 --out gpurun_out/r2y_peer.jsonl > gpurun_out/r2y_peer.log 2>&1
echo peer_rc=$?
timeout 600 python tools/peer_probe.py --gpus 2 --gb 4 --out gpurun_out/r2y_peer.jsonl > gpurun_out/r2y_peer2.log 2>&1
echo peer2_rc=$?
timeout 600 python tools/push_probe.py --gpus 4 --model qwen2.5-7b --tp 2 --only all --out gpurun_out/r2y_push.jsonl > gpurun_out/r2y_push.log 2>&1
echo push_rc=$?
cat gpurun_out/r2y_peer.jsonl
cut -c1-400 gpurun_out/r2y_push.jsonl
tail -3 gpurun_out/r2y_peer.log
