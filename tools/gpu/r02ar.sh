timeout 900 python bench.py > gpurun_out/r02ar_bench.json 2>gpurun_out/r02ar_bench.err; cat gpurun_out/r02ar_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/r02ar_ref.json 2>>gpurun_out/r02ar_bench.err; cat gpurun_out/r02ar_ref.json
