# packed H2D in the drop-in: parity + e2e with / without packing, 4 / 8 / 12 host threads
set -x
mkdir -p gpurun_out
grep -o -w -E "avx512_vbmi2" /proc/cpuinfo | head -1; nproc
timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_o.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_o.log | cut -c1-600
for t in 4 8 12; do
 for pk in 1 0; do
  HJ_PACK_H2D=$pk timeout 200 python bench.py --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 10 --e2e-threads $t 2>>gpurun_out/o.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('pack=$pk thr=$t', d['value'], e['value'], e['pipelined_lane_mpix_s'], e['h2d_bytes_per_step'], e['dense_h2d_bytes_per_step'], e['packed_h2d'], e['bit_exact_vs_oracle'])"
 done
done
for w in 4096p444 4096p422; do
  timeout 200 python bench.py --workload $w --steps 100 --no-cpu-baseline --no-amdahl --e2e-steps 5 --e2e-threads 8 2>>gpurun_out/o.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w pack', d['value'], e['value'], e['h2d_bytes_per_step'], e['dense_h2d_bytes_per_step'], e['bit_exact_vs_oracle'])"
  HJ_PACK_H2D=0 timeout 200 python bench.py --workload $w --steps 100 --no-cpu-baseline --no-amdahl --e2e-steps 5 --e2e-threads 8 2>>gpurun_out/o.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w dense', d['value'], e['value'], e['h2d_bytes_per_step'], e['bit_exact_vs_oracle'])"
done
tail -3 gpurun_out/o.err
