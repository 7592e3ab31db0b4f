# early phase A (HJ_EARLY_A=1: no end-of-step barrier; next step's loads + first
# screen before a deferred barrier) and the static first pixel-item round
# (HJ_GRAB_STATIC=1) vs the shipped kernel; parity suite on the variants first
V=$PWD/paper_1311_5304_b200/variants
for v in early earlyg; do
  HETJPEG_B200_LIB=$V/libhetjpeg_b200_$v.so timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bh_pytest_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/r02bh_pytest_$v.log)"
done
for rep in 1 2; do for v in base grabs early earlyg; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$V/libhetjpeg_b200_$v.so; fi
  for w in 1080p420 4096p444 4096p422; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'])"
  done
  timeout 300 python bench.py --idct islow --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v islow', d['value'], d['roofline']['frac'])"
  unset HETJPEG_B200_LIB
done; done
