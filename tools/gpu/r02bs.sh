# 4:2:0 pixel items of 16 x 1 pixels (HJ_ITEM1ROW=1) vs 16 x 2
V=$PWD/paper_1311_5304_b200/variants
HETJPEG_B200_LIB=$V/libhetjpeg_b200_i1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_gpu_islow.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bs_pytest_i1.log 2>&1; echo "i1 tests: $(tail -1 gpurun_out/r02bs_pytest_i1.log)"
for rep in 1 2; do for v in base i1; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$V/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 24mp420 512p420; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'])"
  done
  timeout 300 python bench.py --idct islow --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v islow', d['value'], d['roofline']['frac'])"
  unset HETJPEG_B200_LIB
done; done
