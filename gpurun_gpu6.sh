for v in base m12 t64 t128; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 4096p444 4096p422; do timeout 120 python bench.py --workload $w --steps 300 --no-cpu-baseline --e2e-steps 1 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"; done
  unset HETJPEG_B200_LIB
done
