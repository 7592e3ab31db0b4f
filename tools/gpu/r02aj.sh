timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in base t128 rows444; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
  for w in 4096p422 4096p444; do
    timeout 200 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'], d['e2e']['bit_exact_vs_oracle'])"
  done
  timeout 200 python bench.py --workload 4096p422 --idct islow --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v islow 4096p422', d['value'], d['roofline']['frac'], d['e2e']['bit_exact_vs_oracle'])"
  unset HETJPEG_B200_LIB
done
