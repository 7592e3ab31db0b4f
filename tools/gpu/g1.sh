set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/microbench/pipes2 > gpurun_out/pipes2.txt 2>&1
cat gpurun_out/pipes2.txt
timeout 600 python bench.py --steps 300 --warmup 10 --no-amdahl > gpurun_out/bench_base.txt 2>&1
tail -c 3000 gpurun_out/bench_base.txt
