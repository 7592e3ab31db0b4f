# Time ablation variants (tools/ablate.sh) on the default workload.
for v in base ${VARIANTS}; do
  if [ $v != base ]; then export HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so; fi
  for w in ${WORKLOADS:-1080p420}; do
    timeout 120 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/ablate.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])" | tee -a gpurun_out/ablate.txt
  done
  unset HETJPEG_B200_LIB
done
