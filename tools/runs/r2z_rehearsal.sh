# round 2, call Z (1 GPU): dress rehearsal of the driver's round-end bench calls with default arguments
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z_build.log 2>&1
t0=$(date +%s); python bench.py > gpurun_out/r2z_bench_default.log 2> gpurun_out/r2z_bench_default.err; rc=$?; echo "elapsed_s=$(( $(date +%s) - t0 ))"
echo bench_rc=$rc
t0=$(date +%s); python bench.py --impl reference > gpurun_out/r2z_bench_ref.log 2> gpurun_out/r2z_bench_ref.err; rc=$?; echo "elapsed_s=$(( $(date +%s) - t0 ))"
echo ref_rc=$rc
grep '^{' gpurun_out/r2z_bench_default.log | tail -1 | cut -c1-300
grep '^{' gpurun_out/r2z_bench_ref.log | tail -1 | cut -c1-300
