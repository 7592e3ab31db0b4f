# grab-ahead of the pixel-item atomics: A/B in one session
VARIANTS="c9 c9rows" WORKLOADS="4096p444" bash tools/gpurun/ablate_run.sh
VARIANTS="c9 c9rows" WORKLOADS="4096p444" bash tools/gpurun/ablate_run.sh
cat gpurun_out/ablate.txt
