# round 2, call R (1 GPU): piece-count sweep of the in-place swap (N=1 bench), two passes
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1
for pass in 1 2; do
  for n in 2 4 8 16; do
    PLEX_SWAP_PIECES=$n timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2r_bench_p${n}_$pass.log 2>&1
  done
done
for f in gpurun_out/r2r_bench_p*.log; do echo $f; grep '^{' $f | tail -1 | cut -c100-200; done
