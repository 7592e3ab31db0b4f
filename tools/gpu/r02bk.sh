# low int16 half via PRMT sign extension + I2FP (HJ_CVT_LO=1) vs I2F.S16 (XU pipe)
V=$PWD/paper_1311_5304_b200/variants
HETJPEG_B200_LIB=$V/libhetjpeg_b200_cvtlo.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_big_hashes.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bk_pytest_cvtlo.log 2>&1; echo "cvtlo tests: $(tail -1 gpurun_out/r02bk_pytest_cvtlo.log)"
for rep in 1 2; do for v in base cvtlo; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$V/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 4096p444 4096p422; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'])"
  done
  unset HETJPEG_B200_LIB
done; done
