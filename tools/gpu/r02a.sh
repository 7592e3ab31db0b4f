set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cat MEASURED_PEAKS.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest_gpu.log 2>&1; tail -5 gpurun_out/r02a_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02a_bench.jsonl 2> gpurun_out/r02a_bench.err; tail -c 2500 gpurun_out/r02a_bench.jsonl
timeout 600 python bench.py --impl reference >> gpurun_out/r02a_bench.jsonl 2>> gpurun_out/r02a_bench.err
timeout 600 python bench.py --impl reference --workload 4096p444 --steps 20 --warmup 3 >> gpurun_out/r02a_bench.jsonl 2>> gpurun_out/r02a_bench.err
HJ_BENCH_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 300 --warmup 5 --no-amdahl --no-cpu-baseline >> gpurun_out/r02a_bench.jsonl 2>> gpurun_out/r02a_bench.err
tail -c 4000 gpurun_out/r02a_bench.jsonl; tail -20 gpurun_out/r02a_bench.err
