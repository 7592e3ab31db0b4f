#!/usr/bin/env bash
# Build the REFERENCE's own native backend (Cython kernels/_native.pyx) from
# its sources under /root/reference, in a scratch copy (/tmp/refbuild; the
# reference tree is read-only and its setup.py writes next to the .pyx).
# Used only by tests/golden/make_golden.py to generate golden fixtures with
# both reference backends.  The build needs Cython + the reference's Python
# package at import time, which does not exist on the GPU box, so the
# reference cannot be the timed CPU baseline there: bench.py's cpu_baseline /
# --impl reference time oracle/render_oracle.c (the bit-exact restatement).
set -e
REF=${REF:-/root/reference/pkg}
OUT=${OUT:-/tmp/refbuild}
[ -d "$REF" ] || { echo "no reference at $REF (skipped)"; exit 0; }
rm -rf "$OUT" && mkdir -p "$OUT" && cp -r "$REF"/. "$OUT"/
cd "$OUT" && python setup.py build_ext --inplace -q > build.log 2>&1 || { echo "reference native build failed (see $OUT/build.log)"; exit 0; }
ls "$OUT"/src/hetjpeg/kernels/_native*.so
