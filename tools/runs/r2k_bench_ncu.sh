# round 2, call K (1 GPU): final N=1 bench + ncu evidence of the same command (launch list)
# and --set full of pack / push on the 3B-shaped bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2k_bench.log 2>&1
echo bench_rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/r02k_plain.log 2>&1; echo plain7_rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pack|push|verify|derive" -c 400 --csv \
  --log-file gpurun_out/r02k_launches.csv $CMD > gpurun_out/r02k_ncu_launches.log 2>&1; echo launches_rc=$?
C3="python bench.py --model qwen2.5-3b --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$C3 > gpurun_out/r02k3_plain.log 2>&1; echo plain3_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 4 -c 2 -o gpurun_out/r02k_pack $C3 > gpurun_out/r02k_ncu_pack.log 2>&1; echo pack_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:push_kernel -c 1 -o gpurun_out/r02k_push $C3 > gpurun_out/r02k_ncu_push.log 2>&1; echo push_rc=$?
grep '^{' gpurun_out/r2k_bench.log | tail -1 | cut -c1-400
grep -o '"roofline": {[^}]*}' gpurun_out/r2k_bench.log
# M5 at D1's FSDP-8 (8 emulated ranks)
timeout 1500 python -m pytest tests/test_gpu_fullsize_configs.py -q -s -m gpu -k m5_ > gpurun_out/r2k_pytest_m5_w8.log 2>&1
echo m5_rc=$?
tail -5 gpurun_out/r2k_pytest_m5_w8.log
grep "M5 trace" gpurun_out/r2k_pytest_m5_w8.log
