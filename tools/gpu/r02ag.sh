timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 2>&1 | tail -1
for w in 1080p420 4096p444 4096p422; do
  timeout 200 python bench.py --workload $w --idct direct --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('direct $w', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"
  HJ_RENDER_TC=1 timeout 200 python bench.py --workload $w --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fast-tc $w', d['value'], d['roofline']['frac'], d['e2e']['bit_exact_vs_oracle'])"
done
