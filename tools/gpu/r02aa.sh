# host Huffman: single-symbol fast table (base) vs + two-symbol AC pair table (pair32), alternating
for i in 1 2 3; do for v in hpair13 huni; do echo -n "$v "; HB_REPS=60 HETJPEG_B200_LIB=$PWD/paper_1311_5304_b200/variants/libhetjpeg_b200_$v.so timeout 300 python tools/microbench/huff_bench.py 2>&1 | tr '\n' '|' | cut -c1-200; echo; done; done
