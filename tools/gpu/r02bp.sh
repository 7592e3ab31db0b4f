# final: smoke (now also idct=direct / islow), default bench line + reference arm
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02bp_bench.json 2>gpurun_out/r02bp_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/r02bp_ref.json 2>>gpurun_out/r02bp_bench.err; echo ref rc=$?
