# end-of-round check: smoke, GPU tests, headline bench + reference arm, direct-mode line (tensor-core kernel)
set -x
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_y.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_y.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_y.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_y.log
O=gpurun_out/r02ah_bench.jsonl; : > $O
timeout 600 python bench.py >> $O 2> gpurun_out/r02ah.err; echo bench rc=$?
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 >> $O 2>> gpurun_out/r02ah.err; echo ref rc=$?
for w in 1080p420 4096p444 4096p422; do
  timeout 300 python bench.py --workload $w --idct direct --steps 300 --no-cpu-baseline --e2e-steps 3 >> $O 2>>gpurun_out/r02ah.err; echo direct $w rc=$?
done
cut -c1-250 $O
