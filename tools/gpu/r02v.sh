# grab-ahead of the pixel-item atomics: A/B in one session
VARIANTS="cols420 cstage0 ldgna0 prmt0 t64c8" WORKLOADS="1080p420" bash tools/gpurun/ablate_run.sh
VARIANTS="cols420 cstage0 ldgna0 prmt0 t64c8" WORKLOADS="1080p420" bash tools/gpurun/ablate_run.sh
cat gpurun_out/ablate.txt
