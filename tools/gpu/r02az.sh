timeout 900 python -m pytest tests/test_gpu_pack.py -q -x -p no:cacheprovider 2>&1 | tail -3
for w in 24mp420 4096p444 4096p422 1080p420 512p420; do
  timeout 600 python bench.py --workload $w --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w', e['value'], e['runs'], e['h2d_bytes_per_step'], e.get('dense_h2d_bytes_per_step'), e['bit_exact_vs_oracle'])"
done
