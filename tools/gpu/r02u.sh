timeout 600 python bench.py --workload 24mp420 --shard rows --steps 100 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02u_rows.jsonl 2>gpurun_out/r02u.err; echo rows1 rc=$?
HJ_BENCH_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --workload 24mp420 --shard rows --steps 100 --no-cpu-baseline --e2e-steps 2 >> gpurun_out/r02u_rows.jsonl 2>>gpurun_out/r02u.err; echo rows2 rc=$?
python -c "
import json
for l in open('gpurun_out/r02u_rows.jsonl'):
    d=json.loads(l); print(d['n_gpus'], d['value'], d['amdahl'])"
