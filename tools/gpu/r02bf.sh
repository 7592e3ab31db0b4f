# HEAD validation (TAG r02bf): GPU tests, smoke, default bench + reference arm,
# launch list of the default bench command, one --set full capture of the 4:2:0 render kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bf_pytest.log 2>&1; tail -1 gpurun_out/r02bf_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bf_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02bf_smoke.log
timeout 900 python bench.py > gpurun_out/r02bf_bench.json 2>gpurun_out/r02bf_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/r02bf_ref.json 2>>gpurun_out/r02bf_bench.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_r02bf.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 \
    -o gpurun_out/prof_r02bf_1080p420 python bench.py --workload 1080p420 --steps 5 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > gpurun_out/ncu_r02bf.log 2>&1; echo ncu full rc=$?
