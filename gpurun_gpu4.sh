timeout 400 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log | cut -c1-600
timeout 60 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for w in 1080p420 4096p444 4096p422 24mp420; do timeout 120 python bench.py --workload $w --steps 300 --no-cpu-baseline --e2e-steps 2 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"; done
export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/libhetjpeg_b200_m3.so
for w in 1080p420 4096p444; do timeout 120 python bench.py --workload $w --steps 300 --no-cpu-baseline --e2e-steps 2 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('m3 $w', d['value'], d['roofline']['frac'], d['idct_screen'])"; done
unset HETJPEG_B200_LIB
timeout 300 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/prof3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full3.log 2>&1; echo ncu rc=$?
