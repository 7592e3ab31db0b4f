# HEAD bench lines (TAG r02bg): headline + reference arm, other configs,
# islow, tensor-core kernel, N=2 ranks sharing the GPU, config 4 row shards, 10k mixed
set -x
mkdir -p gpurun_out
O=gpurun_out/r02bg_bench.jsonl; : > $O
timeout 600 python bench.py >> $O 2> gpurun_out/r02bg.err; echo bench rc=$?
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 >> $O 2>> gpurun_out/r02bg.err; echo ref rc=$?
for w in 512p420 4096p444 4096p422 24mp420; do
  timeout 600 python bench.py --workload $w --steps 300 --e2e-steps 3 >> $O 2>>gpurun_out/r02bg.err; echo $w rc=$?
done
timeout 300 python bench.py --idct islow --steps 300 --e2e-steps 3 >> $O 2>>gpurun_out/r02bg.err
for w in 1080p420 4096p444 4096p422; do timeout 300 python bench.py --workload $w --idct direct --steps 300 --no-cpu-baseline --e2e-steps 3 >> $O 2>>gpurun_out/r02bg.err; done
HJ_BENCH_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 300 --no-cpu-baseline --e2e-steps 3 >> $O 2>>gpurun_out/r02bg.err; echo n2 rc=$?
timeout 600 python bench.py --workload 24mp420 --shard rows --steps 200 --no-cpu-baseline --e2e-steps 3 >> $O 2>>gpurun_out/r02bg.err; echo rows1 rc=$?
HJ_BENCH_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --workload 24mp420 --shard rows --steps 200 --no-cpu-baseline --e2e-steps 3 >> $O 2>>gpurun_out/r02bg.err; echo rows2 rc=$?
timeout 1500 python bench.py --workload mixed --mixed-images 10000 --steps 20 --no-cpu-baseline > gpurun_out/r02bg_mixed10k.jsonl 2>>gpurun_out/r02bg.err; echo mixed rc=$?
cut -c1-200 $O; cut -c1-300 gpurun_out/r02bg_mixed10k.jsonl
tail -5 gpurun_out/r02bg.err
