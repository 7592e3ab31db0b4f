set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_r02i.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02i.log | cut -c1-400
VARIANTS="noscreen nopix neither" WORKLOADS="1080p420 4096p444" bash tools/gpurun/ablate_run.sh
timeout 120 python bench.py --idct islow --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 > gpurun_out/islow.json 2>>gpurun_out/ablate.err; cut -c1-300 gpurun_out/islow.json
cat gpurun_out/ablate.txt
