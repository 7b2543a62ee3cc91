# round 2, call P (1 GPU): piecewise in-place swap -- parity (fast tier + full-size 7B swap) and a same-box
# A/B of the N=1 bench (PLEX_SWAP_PIECES=1 = whole-bucket copies, default 4 pieces)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2p_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" > gpurun_out/r2p_pytest.log 2>&1
echo pytest_rc=$?
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k "swap" > gpurun_out/r2p_pytest_swap7b.log 2>&1
echo swap7b_rc=$?
for i in 1 2; do
  PLEX_SWAP_PIECES=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2p_bench_p1_$i.log 2>&1
  echo p1_rc=$?
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2p_bench_p4_$i.log 2>&1
  echo p4_rc=$?
done
tail -2 gpurun_out/r2p_pytest.log gpurun_out/r2p_pytest_swap7b.log
for f in gpurun_out/r2p_bench_p*.log; do echo $f; grep '^{' $f | tail -1 | cut -c100-260; done
