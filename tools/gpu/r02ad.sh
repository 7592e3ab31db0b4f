for v in base nopix; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
  for idct in fast direct; do
    timeout 200 python bench.py --idct $idct --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $idct', d['value'], d['roofline']['frac'])"
  done
  unset HETJPEG_B200_LIB
done
