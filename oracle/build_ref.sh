#!/usr/bin/env bash
# Build the REFERENCE's own package from its sources under /root/reference
# (read-only; built in scratch copies) into oracle/_ref/ - test
# infrastructure and the CPU baseline arm only, never the product:
#
#   oracle/_ref/shipped/hetjpeg   the reference exactly as its setup.py builds
#                                 it (Cython kernels/_native.pyx, -O3)
#   oracle/_ref/patched/hetjpeg   the same sources with `noexcept` added to the
#                                 13 `cdef ... nogil` helpers (SURVEY.md E2:
#                                 identical arithmetic and bytes; without it
#                                 Cython 3 re-takes the GIL after every call)
#
# oracle/_ref is git-ignored but NOT gpurun-ignored, so both builds travel to
# the GPU box (no /root/reference there).  Used by tests/golden/make_golden.py,
# the drop-in test (tests/test_reference_dropin.py) and bench.py's CPU
# baseline variants.
set -e
REF=${REF:-/root/reference/pkg}
HERE=$(cd "$(dirname "$0")" && pwd)
OUT=${OUT:-$HERE/_ref}
[ -d "$REF" ] || { echo "no reference at $REF (skipped)"; exit 0; }
build() {  # $1 = variant, $2 = patch (0/1)
    local tmp=/tmp/refbuild_$1
    rm -rf "$tmp" && mkdir -p "$tmp" && cp -r "$REF"/. "$tmp"/
    if [ "$2" = 1 ]; then
        sed -i -E 's/\) nogil:$/) noexcept nogil:/' "$tmp/src/hetjpeg/kernels/_native.pyx"
    fi
    (cd "$tmp" && python setup.py build_ext --inplace -q > build.log 2>&1) || {
        echo "reference $1 build failed (see $tmp/build.log)"; return 0; }
    rm -rf "$OUT/$1" && mkdir -p "$OUT/$1"
    cp -r "$tmp/src/hetjpeg" "$OUT/$1/"
    find "$OUT/$1" -name '*.c' -delete
    ls "$OUT/$1"/hetjpeg/kernels/_native*.so
}
build shipped 0
build patched 1
# legacy location used by make_golden.py
rm -rf /tmp/refbuild && cp -r /tmp/refbuild_shipped /tmp/refbuild 2>/dev/null || true
