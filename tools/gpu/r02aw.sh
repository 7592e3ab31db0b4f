for w in 24mp420 4096p444 4096p422 1080p420; do
  for pk in default 1; do
    if [ $pk = 1 ]; then export HJ_PACK_H2D=1; fi
    timeout 600 python bench.py --workload $w --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w pack=$pk', e['value'], e['h2d_bytes_per_step'], e.get('dense_h2d_bytes_per_step'), e['steps'], d['config'].get('images_per_step_per_gpu'))"
    unset HJ_PACK_H2D
  done
done
