python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r02an_smoke.log 2>&1; tail -2 gpurun_out/r02an_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02an_pytest.log 2>&1; tail -3 gpurun_out/r02an_pytest.log
timeout 600 python bench.py > gpurun_out/r02an_bench.json 2>gpurun_out/r02an_bench.err; cat gpurun_out/r02an_bench.json
