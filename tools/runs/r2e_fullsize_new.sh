# round 2, call E (1 GPU): full-size sync parity at M2/M3/M4 (all 8 source ranks
# emulated, rolling masters), the M5 multiplex trace at full size, and the
# pack/unpack in-situ decomposition (tools/pack_insitu.py)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1
timeout 900 python tools/pack_insitu.py --model qwen2.5-7b --out gpurun_out/r2e_pack_insitu.jsonl > gpurun_out/r2e_pack_insitu.log 2>&1
echo insitu_rc=$?
timeout 4200 python -m pytest tests/test_gpu_fullsize_configs.py -v -m gpu --durations=0 \
  -k "m2_qwen7b_fsdp8 or m3_qwen32b_fsdp8 or m4_qwen3_30b_a3b_fsdp8 or m5_" > gpurun_out/r2e_pytest_fullsize.log 2>&1
echo pytest_rc=$?
tail -30 gpurun_out/r2e_pytest_fullsize.log
cat gpurun_out/r2e_pack_insitu.jsonl | cut -c1-300
# ncu evidence: launch list of the N=1 bench command itself (7B), then --set full
# captures of pack / push on the 3B-shaped bench (ncu cannot back up the 7B job's
# 106.6 GB for kernel replay; same kernels, same 2 GiB buckets)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/r02g_plain.log 2>&1; echo plain7_rc=$?
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pack|push|verify|derive" -c 400 --csv \
  --log-file gpurun_out/r02g_launches.csv $CMD > gpurun_out/r02g_ncu_launches.log 2>&1; echo launches_rc=$?
C3="python bench.py --model qwen2.5-3b --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$C3 > gpurun_out/r02f_plain.log 2>&1; echo plain3_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 4 -c 2 -o gpurun_out/r02f_pack $C3 > gpurun_out/r02f_ncu_pack.log 2>&1; echo pack_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:push_kernel -c 1 -o gpurun_out/r02f_push $C3 > gpurun_out/r02f_ncu_push.log 2>&1; echo push_rc=$?
ls -la gpurun_out/ | tail -20
