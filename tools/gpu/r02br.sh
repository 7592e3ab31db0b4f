# 4:2:0 with 256-thread CTAs x 2 per SM (strips of 84 MCUs) vs 128 x 4 (42 MCUs)
V=$PWD/paper_1311_5304_b200/variants
HETJPEG_B200_LIB=$V/libhetjpeg_b200_t256.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_gpu_islow.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02br_pytest_t256.log 2>&1; echo "t256 tests: $(tail -1 gpurun_out/r02br_pytest_t256.log)"
for rep in 1 2; do for v in base t256; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$V/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 24mp420 512p420; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'])"
  done
  timeout 300 python bench.py --idct islow --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v islow', d['value'], d['roofline']['frac'])"
  unset HETJPEG_B200_LIB
done; done
