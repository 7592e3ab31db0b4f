for rep in 1 2; do for v in old new; do for w in 512p420 1080p420; do
  if [ $v = old ]; then
    timeout 600 python -c "
import sys, runpy
import paper_1311_5304_b200._lib as L
L.ptr = lambda a: a.ctypes.data
sys.argv = ['bench.py', '--workload', '$w', '--steps', '50', '--no-cpu-baseline', '--no-amdahl', '--e2e-steps', '20']
runpy.run_path('bench.py', run_name='__main__')" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v $w', e['value'], e['runs'])"
  else
    timeout 600 python bench.py --workload $w --steps 50 --no-cpu-baseline --no-amdahl --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v $w', e['value'], e['runs'])"
  fi
done; done; done
