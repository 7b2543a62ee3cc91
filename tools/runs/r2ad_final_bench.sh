# round 2, call AD (1 GPU): N=1 bench at the final commit
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ad_build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2ad_bench.log 2>&1
echo bench_rc=$?
grep '^{' gpurun_out/r2ad_bench.log | tail -1 | cut -c1-300
