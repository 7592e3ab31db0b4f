# static first pixel-item round in the reference-mode kernels (HJ_GRAB_STATIC default 1):
# GPU suite, racecheck / synccheck of the render kernels, bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bi_pytest.log 2>&1; tail -1 gpurun_out/r02bi_pytest.log
for tool in racecheck synccheck; do
  for t in test_gpu_parity test_gpu_tc; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/$t.py -m gpu -x -q -p no:cacheprovider \
      -k "not full_size and not big and not 4096 and not 24 and not exhaustive" > gpurun_out/r02bi_san_${tool}_$t.txt 2>&1
    echo "$tool $t rc=$? $(grep -E 'passed|failed' gpurun_out/r02bi_san_${tool}_$t.txt | tail -1) $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r02bi_san_${tool}_$t.txt | tail -1)"
  done
done
for w in 1080p420 4096p444 4096p422 24mp420 512p420; do
  timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'])"
done
timeout 300 python bench.py --idct islow --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('islow', d['value'], d['roofline']['frac'])"
timeout 300 python bench.py --idct direct --steps 300 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('direct', d['value'], d['roofline']['frac'])"
timeout 600 python bench.py --workload mixed --mixed-images 96 --steps 20 --no-cpu-baseline --no-amdahl --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mixed', d['value'], d['roofline']['frac'])"
