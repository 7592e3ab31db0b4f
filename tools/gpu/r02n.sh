# L2-resident vs streaming: is the v3 kernel's time memory- or issue-bound?
for b in 128 16 8; do
  for v in base neither; do
    if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
    timeout 120 python bench.py --batch $b --steps 400 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/n.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v batch $b', d['value'], d['roofline']['frac'], d['ms_per_step'])"
    unset HETJPEG_B200_LIB
  done
done
