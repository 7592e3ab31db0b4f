set -x
free -g | head -2; nproc
timeout 600 python -m pytest tests/test_stream.py -x -q > gpurun_out/r02e_stream.log 2>&1; tail -5 gpurun_out/r02e_stream.log
timeout 1500 python tools/profile_b200.py --out gpurun_out/b200_profile_r02.json > gpurun_out/r02e_profile.log 2>&1; tail -3 gpurun_out/r02e_profile.log
cp gpurun_out/b200_profile_r02.json profiles/b200_profile.json 2>/dev/null
timeout 900 python bench.py --workload mixed --mixed-images 10000 --steps 20 --warmup 3 > gpurun_out/r02e_mixed.jsonl 2> gpurun_out/r02e_mixed.err; tail -c 3500 gpurun_out/r02e_mixed.jsonl; tail -5 gpurun_out/r02e_mixed.err
