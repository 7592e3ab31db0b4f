for w in 1080p420 4096p444 4096p422; do
  timeout 300 python bench.py --workload $w --idct direct --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/x.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w direct', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:render_tc -s 3 -c 1 -o gpurun_out/prof_r02x python bench.py --idct direct --steps 5 --warmup 3 --no-cpu-baseline --no-amdahl --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
