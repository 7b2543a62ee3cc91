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
