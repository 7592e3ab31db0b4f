HJ_BENCH_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 200 > gpurun_out/r02av_n2.json 2> gpurun_out/r02av_n2.err; echo rc=$?; cat gpurun_out/r02av_n2.json | cut -c1-600
HJ_BENCH_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > gpurun_out/r02av_n2_ref.json 2>> gpurun_out/r02av_n2.err; echo rc=$?; cat gpurun_out/r02av_n2_ref.json | cut -c1-300
tail -3 gpurun_out/r02av_n2.err
