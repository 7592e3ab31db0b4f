# final-state ncu captures (TAG r02as): launch list of the default bench command and one
# --set full capture of the render kernel per workload
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_r02as.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
for w in 1080p420 4096p444 4096p422; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 \
    -o gpurun_out/prof_r02as_$w python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > gpurun_out/ncu_$w.log 2>&1; echo ncu $w rc=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 \
    -o gpurun_out/prof_r02as_islow python bench.py --idct islow --steps 5 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > gpurun_out/ncu_islow.log 2>&1; echo ncu islow rc=$?
ls -la gpurun_out/*.ncu-rep
