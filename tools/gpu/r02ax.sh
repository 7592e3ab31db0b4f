for rep in 1 2 3; do for t in 8 12; do
  timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 20 --e2e-threads $t 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('t$t', e['value'])"
done; done
for rep in 1 2; do
  timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('s10', e['value'])"
done
cat /proc/loadavg; nproc
