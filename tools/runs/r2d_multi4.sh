# round 2, call D (4 GPUs): multi-GPU parity (group executor, collectives), bench N=2/4,
# push probe (single process over 4 GPUs) + its ncu capture with DRAM and NVLink counters,
# sync / moe scenarios with clocks
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2d_topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_multi.py -v -m gpu --durations=0 > gpurun_out/r2d_pytest_multi.log 2>&1
echo pytest_rc=$?
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2d_bench_n2.log 2>&1
echo bench2_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2d_bench_n4.log 2>&1
echo bench4_rc=$?
for only in all row col; do
  timeout 600 python tools/push_probe.py --gpus 4 --model qwen2.5-7b --tp 2 --only $only --out gpurun_out/r2d_push_probe.jsonl > gpurun_out/r2d_probe_$only.log 2>&1
  echo probe_${only}_rc=$?
done
timeout 600 python tools/push_probe.py --gpus 4 --model qwen2.5-32b --tp 4 --only row --out gpurun_out/r2d_push_probe.jsonl > gpurun_out/r2d_probe_32b_row.log 2>&1
timeout 600 python tools/push_probe.py --gpus 4 --model qwen2.5-32b --tp 4 --only all --out gpurun_out/r2d_push_probe.jsonl > gpurun_out/r2d_probe_32b_all.log 2>&1
echo probe32_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29513 tools/scenarios.py --scenario sync --gpus 4 --steps 5 --warmup 2 --out gpurun_out/r2d_scen.jsonl > gpurun_out/r2d_scen_sync.log 2>&1
echo sync_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29514 tools/scenarios.py --scenario sync --gpus 4 --model qwen2.5-7b --tp 2 --steps 5 --warmup 2 --out gpurun_out/r2d_scen.jsonl > gpurun_out/r2d_scen_sync7.log 2>&1
echo sync7_rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29515 tools/scenarios.py --scenario moe --gpus 4 --steps 5 --warmup 2 --out gpurun_out/r2d_scen.jsonl > gpurun_out/r2d_scen_moe.log 2>&1
echo moe_rc=$?
# ncu: same command line just exited 0 above without ncu (probe_row / probe_all)
P="python tools/push_probe.py --gpus 4 --model qwen2.5-7b --tp 2 --steps 1 --warmup 0"
$P --only row > gpurun_out/r2d_ncu_plain_row.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:push_kernel --csv --log-file gpurun_out/r2d_ncu_push_row.csv $P --only row > gpurun_out/r2d_ncu_row.log 2>&1
echo ncu_row_rc=$?
$P --only all > gpurun_out/r2d_ncu_plain_all.log 2>&1 && \
ncu --set full --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
    --clock-control none --import-source on -k regex:push_kernel -c 4 -o gpurun_out/r2d_push_full $P --only all > gpurun_out/r2d_ncu_all.log 2>&1
echo ncu_all_rc=$?
tail -3 gpurun_out/r2d_pytest_multi.log
tail -c 1500 gpurun_out/r2d_bench_n4.log
cat gpurun_out/r2d_push_probe.jsonl | cut -c1-400
