# shipped per-subsampling static item rounds (4:4:4: 2, else 1): GPU suite + kernel lines
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bn_pytest.log 2>&1; tail -1 gpurun_out/r02bn_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for w in 1080p420 4096p444 4096p422 24mp420 512p420; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'])"
done
for w in 1080p420 4096p444 4096p422; do
timeout 300 python bench.py --workload $w --idct direct --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('direct $w', d['value'], d['roofline']['frac'])"
done
timeout 300 python bench.py --idct islow --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('islow', d['value'], d['roofline']['frac'])"
timeout 600 python bench.py --workload mixed --mixed-images 96 --steps 20 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mixed', d['value'], d['roofline']['frac'])"
