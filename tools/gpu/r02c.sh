set -x
timeout 900 python -m pytest tests/test_gpu_islow.py -x -q > gpurun_out/r02c_islow.log 2>&1; tail -25 gpurun_out/r02c_islow.log
