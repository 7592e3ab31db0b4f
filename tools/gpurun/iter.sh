# Iteration loop: GPU parity tests, bench lines, one ncu --set full capture.
#   TAG=v3c bash tools/gpurun/iter.sh
TAG=${TAG:-iter}
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log | cut -c1-400
VARIANTS="${VARIANTS}" WORKLOADS="${WORKLOADS:-1080p420 4096p444 4096p422}" bash tools/gpurun/ablate_run.sh
if [ -z "$SKIP_NCU" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
fi
