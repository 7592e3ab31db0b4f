for rep in 1 2 3; do for v in base blk; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
  for t in 8 12 16; do
  timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 20 --e2e-threads $t 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v t$t', e['value'])"
  done
  unset HETJPEG_B200_LIB
done; done
