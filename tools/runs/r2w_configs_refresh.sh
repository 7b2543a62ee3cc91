# round 2, call W (4 GPUs): configs[2] optimizer offload at k = 1 / 2 / 4 (rank r of the 32B FSDP-8 plan),
# configs[3] MoE EP-4 sync + per-expert units, NEXT-2 ZeRO-2 dedup at 4 GPUs -- final code, with clocks
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python tools/scenarios.py --scenario optim --gpus 1 --out gpurun_out/r2w_scen.jsonl > gpurun_out/r2w_optim1.log 2>&1
echo optim1_rc=$?
timeout 900 $TR --nproc-per-node 2 --master-port 29561 tools/scenarios.py --scenario optim --gpus 2 --out gpurun_out/r2w_scen.jsonl > gpurun_out/r2w_optim2.log 2>&1
echo optim2_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29562 tools/scenarios.py --scenario optim --gpus 4 --out gpurun_out/r2w_scen.jsonl > gpurun_out/r2w_optim4.log 2>&1
echo optim4_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29563 tools/scenarios.py --scenario moe --gpus 4 --steps 5 --warmup 2 --out gpurun_out/r2w_scen.jsonl > gpurun_out/r2w_moe4.log 2>&1
echo moe4_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29564 tools/scenarios.py --scenario zero2 --gpus 4 --out gpurun_out/r2w_scen.jsonl > gpurun_out/r2w_zero2.log 2>&1
echo zero2_rc=$?
cut -c1-700 gpurun_out/r2w_scen.jsonl
