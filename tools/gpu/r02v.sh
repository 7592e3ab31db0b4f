# grab-ahead of the pixel-item atomics: A/B in one session
VARIANTS="minw3 minw4 minw8 minw420_3" WORKLOADS="1080p420 4096p444 4096p422" bash tools/gpurun/ablate_run.sh
VARIANTS="minw3 minw4 minw8 minw420_3" WORKLOADS="1080p420 4096p444 4096p422" bash tools/gpurun/ablate_run.sh
cat gpurun_out/ablate.txt
