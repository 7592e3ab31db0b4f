set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02f_pytest_gpu.log 2>&1; tail -5 gpurun_out/r02f_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r02f_bench.jsonl 2> gpurun_out/r02f_bench.err; tail -c 1500 gpurun_out/r02f_bench.jsonl
timeout 900 python bench.py --workload mixed --mixed-images 10000 --steps 20 --warmup 3 > gpurun_out/r02f_mixed.jsonl 2> gpurun_out/r02f_mixed.err; tail -c 2500 gpurun_out/r02f_mixed.jsonl; tail -3 gpurun_out/r02f_mixed.err
