set -x
VARIANTS="noscreen nopix neither" WORKLOADS="1080p420 4096p444" bash tools/gpurun/ablate_run.sh
cat gpurun_out/ablate.txt
