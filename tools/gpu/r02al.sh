# mixed pool kernel rate: 4:2:2 configuration old (6 CTAs, column screen) vs new (8 CTAs, row screen), alternating
for i in 1 2; do
for v in base old422; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
  timeout 600 python bench.py --workload mixed --mixed-images 96 --steps 20 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v mixed', d['value'], d['roofline']['frac'])"
  unset HETJPEG_B200_LIB
done
done
