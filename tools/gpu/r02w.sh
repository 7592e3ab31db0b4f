set -x
timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_w.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_w.log | cut -c1-800
for w in 1080p420 4096p444 4096p422; do
 for m in def 0; do
  if [ $m = def ]; then unset HJ_RENDER_TC; else export HJ_RENDER_TC=$m; fi
  timeout 300 python bench.py --workload $w --idct direct --steps 100 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/w.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w direct tc=$m', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"
 done
done
unset HJ_RENDER_TC
tail -3 gpurun_out/w.err
