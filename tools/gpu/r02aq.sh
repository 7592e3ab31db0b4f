for rep in 1 2; do for t in 8 12 16 6; do
  timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 20 --e2e-threads $t 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('threads $t', e['value'], e['h2d_bytes_per_step'], e['packed_h2d'])"
done; done
nproc; lscpu | grep -E "Model name|^CPU\(s\)|NUMA node\(s\)"
