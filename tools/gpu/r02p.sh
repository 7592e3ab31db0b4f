# chunk-pipelined packed H2D: parity, e2e auto vs dense across host threads and workloads
set -x
mkdir -p gpurun_out
#timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_p.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_p.log | cut -c1-600
for w in 1080p420 4096p444 4096p422; do
 for t in 4 8; do
  for pk in auto 0; do
   if [ $pk = auto ]; then unset HJ_PACK_H2D; else export HJ_PACK_H2D=$pk; fi
   timeout 300 python bench.py --workload $w --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 5 --e2e-threads $t 2>>gpurun_out/p.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w thr=$t pack=$pk', e['value'], e['pipelined_lane_mpix_s'], e['h2d_bytes_per_step'], e['dense_h2d_bytes_per_step'], e['packed_h2d'], e['bit_exact_vs_oracle'])"
  done
 done
done
unset HJ_PACK_H2D
tail -3 gpurun_out/p.err
