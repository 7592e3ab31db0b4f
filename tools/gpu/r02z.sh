# mixed pool kernel: launch list (per-family kernels) + per-family timing
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --clock-control none -c 12 --csv \
    --log-file gpurun_out/launches_mixed.csv python bench.py --workload mixed --mixed-images 96 --steps 3 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_summary.py --launches gpurun_out/launches_mixed.csv
