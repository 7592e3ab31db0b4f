for rep in 1 2 3; do for pk in 0 default; do
  if [ $pk = 0 ]; then export HJ_PACK_H2D=0; fi
  timeout 600 python bench.py --workload 24mp420 --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('24mp pack=$pk', e['value'], e['runs'], e['h2d_bytes_per_step'])"
  unset HJ_PACK_H2D
done; done
