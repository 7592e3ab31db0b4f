# static pixel-item rounds per warp and step: 1 (shipped) vs 2 / 3 (HJ_GRAB_STATIC=2/3)
V=$PWD/paper_1311_5304_b200/variants
for v in gs2 gs3; do
HETJPEG_B200_LIB=$V/libhetjpeg_b200_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_gpu_tc.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bm_pytest_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/r02bm_pytest_$v.log)"
done
for rep in 1 2; do for v in base gs2 gs3; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$V/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 4096p444 4096p422; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'])"
  done
  unset HETJPEG_B200_LIB
done; done
