# round 2, call Q (1 GPU): copy-engine timeline of the bench's N=1 in-place swap (7B, 2 GiB buckets),
# whole-bucket copies (PLEX_SWAP_PIECES=1) vs 4 pieces, alternating; then 3 more bench A/B pairs
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q_build.log 2>&1
for i in 1 2; do
  PLEX_SWAP_PIECES=1 timeout 900 python tools/timeline.py --model qwen2.5-7b --bucket-mb 2048 --swap --out gpurun_out/r2q_timeline.txt > gpurun_out/r2q_tl_p1_$i.log 2>&1
  echo tl1_rc=$?
  timeout 900 python tools/timeline.py --model qwen2.5-7b --bucket-mb 2048 --swap --out gpurun_out/r2q_timeline.txt > gpurun_out/r2q_tl_p4_$i.log 2>&1
  echo tl4_rc=$?
done
for i in 3 4 5; do
  PLEX_SWAP_PIECES=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2q_bench_p1_$i.log 2>&1
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2q_bench_p4_$i.log 2>&1
done
grep '^{"model' gpurun_out/r2q_timeline.txt | cut -c1-900
for f in gpurun_out/r2q_bench_p*.log; do echo $f; grep '^{' $f | tail -1 | cut -c100-200; done
