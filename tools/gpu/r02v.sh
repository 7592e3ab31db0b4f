# grab-ahead of the pixel-item atomics: A/B in one session
VARIANTS="unroll nospecial" WORKLOADS="1080p420 4096p444 4096p422" bash tools/gpurun/ablate_run.sh
VARIANTS="unroll nospecial" WORKLOADS="1080p420 4096p444 4096p422" bash tools/gpurun/ablate_run.sh
cat gpurun_out/ablate.txt
