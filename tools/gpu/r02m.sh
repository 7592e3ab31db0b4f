set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_m.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_m.log | cut -c1-600
timeout 120 python bench.py --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/bench_m.err | cut -c1-400
