# One gpurun call: smoke, GPU parity tests, bench lines for every workload,
# ncu launch list + one --set full capture of the render kernel.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpurun/round.sh'
# Optional env: TAG (profile name suffix), SKIP_TESTS=1, SKIP_NCU=1.
set -x
TAG=${TAG:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
  tail -4 gpurun_out/pytest_gpu.log | cut -c1-800
fi
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 200 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
: > gpurun_out/bench_other.json
for w in 512p420 4096p444 4096p422 24mp420 mixed; do
  timeout 200 python bench.py --workload $w --steps 300 --no-cpu-baseline --e2e-steps 3 >> gpurun_out/bench_other.json 2>>gpurun_out/bench.err
done
cut -c1-400 gpurun_out/bench_other.json
if [ -z "$SKIP_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
  tail -3 gpurun_out/ncu_full.log
fi
