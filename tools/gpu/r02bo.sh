# tensor-core kernel back to one static item round at 4:4:4: GPU suite + kernel lines
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bo_pytest.log 2>&1; tail -1 gpurun_out/r02bo_pytest.log
for w in 1080p420 4096p444 4096p422; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'])"
  timeout 300 python bench.py --workload $w --idct direct --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('direct $w', d['value'], d['roofline']['frac'])"
done
