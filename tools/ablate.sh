# Build ablation variants of the library (timing studies only; wrong bytes):
#   bash tools/ablate.sh NAME "-DFLAG ..."  -> paper_1311_5304_b200/variants/libhetjpeg_b200_NAME.so
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1311_5304_b200/variants
C=paper_1311_5304_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-ffp-contract=off -shared $2 \
  -o paper_1311_5304_b200/variants/libhetjpeg_b200_$1.so $C/hj_render.cu $C/hj_blockops.cu $C/hj_api.cu $C/hj_huffman.cpp $C/hj_sched.cpp $C/hj_pack.cpp
