# tensor-core kernel: N=192 units (1 TMEM buffer, 4 units / step) vs N=96 x 2 (default); parity first
HJ_RENDER_TC=1 HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_tc64.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 900 2>&1 | tail -1
HJ_RENDER_TC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 900 2>&1 | tail -1
for v in base tc64; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 4096p444 4096p422; do
    timeout 200 python bench.py --workload $w --idct direct --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v direct $w', d['value'], d['roofline']['frac'], d['e2e']['bit_exact_vs_oracle'])"
  done
  unset HETJPEG_B200_LIB
done
