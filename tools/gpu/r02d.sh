# round-2 measurements: islow mode lines + ncu of the islow 4:2:0 kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for w in 1080p420 4096p444 4096p422 512p420 24mp420; do
  timeout 600 python bench.py --workload $w --idct islow --steps 500 --warmup 10 $( [ $w = 1080p420 ] || echo --no-amdahl ) >> gpurun_out/r02d_bench.jsonl 2>> gpurun_out/r02d_bench.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02d_launches_islow.csv python bench.py --idct islow --steps 20 --warmup 3 --no-amdahl --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/prof_r02d_islow420 python bench.py --idct islow --steps 5 --warmup 3 --no-amdahl --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
echo ncu rc=$?
tail -c 3000 gpurun_out/r02d_bench.jsonl
