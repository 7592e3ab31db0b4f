# final-tree check: GPU suite, smoke, the N=2 path (two ranks sharing the one GPU) and its reference arm
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bq_pytest.log 2>&1; tail -1 gpurun_out/r02bq_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
HJ_BENCH_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 300 --no-cpu-baseline --e2e-steps 3 > gpurun_out/r02bq_n2.json 2>gpurun_out/r02bq_n2.err; echo n2 rc=$?
HJ_BENCH_SHARE_DEVICE=1 timeout 600 python bench.py --impl reference --gpus 2 > gpurun_out/r02bq_n2_ref.json 2>>gpurun_out/r02bq_n2.err; echo n2 ref rc=$?
cut -c1-300 gpurun_out/r02bq_n2.json gpurun_out/r02bq_n2_ref.json
