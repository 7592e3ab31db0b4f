# final-state captures (TAG r02bj, static first item round): default bench line + reference arm,
# launch list of the default bench command, ncu --set full of the 1080p 4:2:0 / 4096^2 4:4:4 / 4:2:2 render kernels
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02bj_bench.json 2>gpurun_out/r02bj_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/r02bj_ref.json 2>>gpurun_out/r02bj_bench.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_r02bj.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
for w in 1080p420 4096p444 4096p422; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 \
    -o gpurun_out/prof_r02bj_$w python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > gpurun_out/ncu_r02bj_$w.log 2>&1; echo ncu $w rc=$?
done
