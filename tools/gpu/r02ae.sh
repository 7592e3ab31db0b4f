# tensor-core kernel: N=48 units x 5 TMEM buffers (default build) vs N=96 x 2 (tc32); direct and fast (HJ_RENDER_TC=1)
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -m gpu -x -q -k "tc or direct or golden" --timeout 900 2>&1 | tail -2
for v in base tc32; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 4096p444 4096p422; do
    timeout 200 python bench.py --workload $w --idct direct --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v direct $w', d['value'], d['roofline']['frac'], d['e2e']['bit_exact_vs_oracle'])"
    HJ_RENDER_TC=1 timeout 200 python bench.py --workload $w --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v fast-tc $w', d['value'], d['roofline']['frac'], d['e2e']['bit_exact_vs_oracle'])"
  done
  unset HETJPEG_B200_LIB
done
