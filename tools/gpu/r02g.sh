set -x
timeout 900 python bench.py --workload 24mp420 --shard rows --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/r02g_rows1.jsonl 2> gpurun_out/r02g.err; tail -c 1800 gpurun_out/r02g_rows1.jsonl
HJ_BENCH_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --workload 24mp420 --shard rows --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/r02g_rows2.jsonl 2>> gpurun_out/r02g.err; tail -c 1800 gpurun_out/r02g_rows2.jsonl
for w in 4096p444 4096p422; do
timeout 1200 python bench.py --workload $w --steps 100 --warmup 5 --no-amdahl --cpu-variants > gpurun_out/r02g_cpuvar_$w.jsonl 2>> gpurun_out/r02g.err; tail -c 2500 gpurun_out/r02g_cpuvar_$w.jsonl
done
tail -5 gpurun_out/r02g.err
