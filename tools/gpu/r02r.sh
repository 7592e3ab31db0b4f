# round-2 measurement of the shipped state (TAG=r02r): smoke, GPU tests, all bench
# workloads (+ islow), reference arm, ncu launch list + one --set full capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_r.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_r.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_r.log
timeout 400 python bench.py > gpurun_out/bench_r.jsonl 2> gpurun_out/bench_r.err; echo bench rc=$?
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 >> gpurun_out/bench_r.jsonl 2>> gpurun_out/bench_r.err; echo ref rc=$?
for w in 512p420 4096p444 4096p422 24mp420; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --e2e-steps 3 >> gpurun_out/bench_r.jsonl 2>>gpurun_out/bench_r.err
done
timeout 300 python bench.py --idct islow --steps 300 --no-cpu-baseline --e2e-steps 3 >> gpurun_out/bench_r.jsonl 2>>gpurun_out/bench_r.err
HJ_RENDER_TC=1 timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 3 >> gpurun_out/bench_r.jsonl 2>>gpurun_out/bench_r.err
cut -c1-300 gpurun_out/bench_r.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_r02r.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 \
    -o gpurun_out/prof_r02r python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/bench_r.err
