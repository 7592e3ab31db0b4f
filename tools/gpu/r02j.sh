# first light of the tensor-core screen: smoke, GPU parity, bench TC vs SIMT
set -x
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_j.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke_j.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_j.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_j.log | cut -c1-600
for w in 1080p420 4096p444 4096p422; do
  timeout 120 python bench.py --workload $w --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/bench_j.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tc $w', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"
  HJ_RENDER_SIMT=1 timeout 120 python bench.py --workload $w --steps 200 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>>gpurun_out/bench_j.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('simt $w', d['value'], d['roofline']['frac'], d['idct_screen'], d['e2e']['bit_exact_vs_oracle'])"
done
tail -5 gpurun_out/bench_j.err
