set -x
mkdir -p gpurun_out
timeout 60 ./tools/microbench/tc_lat_probe > gpurun_out/tc_lat2.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_l.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_l.log | cut -c1-600
for w in 1080p420 4096p444 4096p422; do
  timeout 120 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/bench_l.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tc $w', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:render_tc -s 3 -c 1 -o gpurun_out/prof_r02l python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
cat gpurun_out/tc_lat2.txt
