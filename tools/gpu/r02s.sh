for w in 512p420 24mp420 1080p420; do
 for pk in auto 0; do
   if [ $pk = auto ]; then unset HJ_PACK_H2D; else export HJ_PACK_H2D=$pk; fi
   timeout 300 python bench.py --workload $w --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 5 2>>gpurun_out/s.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w pack=$pk', d['config']['images_per_step_per_gpu'], e['value'], e['pipelined_lane_mpix_s'], e['h2d_bytes_per_step'], e['dense_h2d_bytes_per_step'], e['bit_exact_vs_oracle'])"
 done
done
unset HJ_PACK_H2D
