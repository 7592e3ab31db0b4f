# compute-sanitizer on the render kernels (v3 and the tensor-core v4): memcheck, racecheck, synccheck
cat > /tmp/san.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1311_5304_b200 import entropy, parser
from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
from paper_1311_5304_b200.perf_model import qtable_stack
from paper_1311_5304_b200.synth import synth_jpeg
from oracle import oracle
for (w, h, sub) in [(200, 130, "420"), (136, 72, "422"), (120, 64, "444")]:
    blob = synth_jpeg(w, h, 90, sub, seed=1)
    p = parser.parse_stream(blob); co, _ = entropy.decode_all(p, blob); g = co.geometry; q = qtable_stack(p)
    for fast in (True, False):
        px = alloc_pixels(w, h); render_rows(co, q, px, 0, g.mcu_rows, fast=fast)
        want = oracle.render(co.y_blocks, co.cb_blocks, co.cr_blocks, q, w, h, {"444": 0, "422": 1, "420": 2}[sub], fast)
        assert np.array_equal(px.data, want), (w, h, sub, fast)
print("ok")
PY
for tool in memcheck racecheck synccheck; do
  for tc in 0 1; do
    HJ_RENDER_TC=$tc timeout 900 compute-sanitizer --tool $tool --print-limit 5 python /tmp/san.py > gpurun_out/san_${tool}_${tc}.txt 2>&1; echo "$tool tc=$tc rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^ok" gpurun_out/san_${tool}_${tc}.txt | head -3
  done
done
