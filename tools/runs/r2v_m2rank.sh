# round 2, call V (4 GPUs): the M2 per-GPU workload (rank r of the 7B FSDP-8 -> TP-2xDP-4 plan, duplex switch
# through the group executor) with k = 1 / 2 / 4 GPUs switching at once
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2v_topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python tools/scenarios.py --scenario m2rank --gpus 1 --steps 6 --warmup 2 --out gpurun_out/r2v_m2rank.jsonl > gpurun_out/r2v_k1.log 2>&1
echo k1_rc=$?
timeout 900 $TR --nproc-per-node 2 --master-port 29551 tools/scenarios.py --scenario m2rank --gpus 2 --steps 6 --warmup 2 --out gpurun_out/r2v_m2rank.jsonl > gpurun_out/r2v_k2.log 2>&1
echo k2_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29552 tools/scenarios.py --scenario m2rank --gpus 4 --steps 6 --warmup 2 --out gpurun_out/r2v_m2rank.jsonl > gpurun_out/r2v_k4.log 2>&1
echo k4_rc=$?
cat gpurun_out/r2v_m2rank.jsonl
tail -3 gpurun_out/r2v_k4.log
