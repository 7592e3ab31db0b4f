"""Rigorous first-order error constants for the FP32 screen of the AAN IDCT
(csrc/hj_render.cu `screen_block`).  Emits csrc/hj_screen.h.

Model: the screen evaluates the reference's AAN
DAG (_native.pyx:321-388) in IEEE binary32 with round-to-nearest, FFMA at
tmp12 / t10 / t12 (one rounding), binary32 constants, inputs
x_i = fl(fl(float(c_i)) * fl(q_i*pre_i)).  For every output o

  |o_fp32 - o_exact| <= u * sum_i K[o,i] |x_i| + O(u^2),   u = 2^-24,

where K[o,i] = sum_v |do/dv| |dv/dx_i| over every rounded node v (each
binary op / FFMA), plus the binary32 rounding of each multiplier constant
(|do/dv| |c| |da/dx_i| at v = c*a) and of the inputs (2 |do/dx_i|).  The
kernel uses Kmax_i = max_o K[o,i]; the float64 reference deviates from exact
real arithmetic by the same expression with u = 2^-53, folded into SAFETY.
"""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SQRT2, ROT, ROT_P, ROT_M = 1.414213562, 1.847759065, 1.082392200, 2.613125930


class Lin:
    """Linear form over the 64 inputs plus a list of (node coefficient
    vector, kind) for error accounting is done by the tracer below."""


def trace():
    # Each value is a 64-vector of coefficients (the DAG is linear).
    nodes = []      # (coef_vec, const_err_vec or None, name)

    def rnd(v, const_term=None):
        nodes.append((v, const_term))
        return (v, len(nodes) - 1)

    def val(a):
        return a[0]

    def aan(d):
        d0, d1, d2, d3, d4, d5, d6, d7 = d
        add = lambda a, b: rnd(val(a) + val(b))          # noqa: E731
        sub = lambda a, b: rnd(val(a) - val(b))          # noqa: E731
        tmp10 = add(d0, d4); tmp11 = sub(d0, d4); tmp13 = add(d2, d6)
        a = sub(d2, d6)
        tmp12 = rnd(SQRT2 * val(a) - val(tmp13), np.abs(SQRT2 * val(a)))      # FFMA
        e0 = add(tmp10, tmp13); e3 = sub(tmp10, tmp13); e1 = add(tmp11, tmp12); e2 = sub(tmp11, tmp12)
        z13 = add(d5, d3); z10 = sub(d5, d3); z11 = add(d1, d7); z12 = sub(d1, d7)
        t7 = add(z11, z13); b = sub(z11, z13)
        t11 = rnd(SQRT2 * val(b), np.abs(SQRT2 * val(b)))
        c = add(z10, z12)
        z5 = rnd(ROT * val(c), np.abs(ROT * val(c)))
        t10 = rnd(ROT_P * val(z12) - val(z5), np.abs(ROT_P * val(z12)))         # FFMA
        t12 = rnd(-ROT_M * val(z10) + val(z5), np.abs(ROT_M * val(z10)))       # FFMA
        t6 = sub(t12, t7); t5 = sub(t11, t6); t4 = add(t10, t5)
        return [add(e0, t7), add(e1, t6), add(e2, t5), sub(e3, t4),
                add(e3, t4), sub(e2, t5), sub(e1, t6), sub(e0, t7)]

    x = [(np.eye(64)[i], None) for i in range(64)]
    g = [[None] * 8 for _ in range(8)]
    for c in range(8):
        col = aan([x[r * 8 + c] for r in range(8)])
        for r in range(8):
            g[r][c] = col[r]
    out = []
    for r in range(8):
        out += aan(g[r])
    return nodes, out


def influence(nodes, out):
    """|d out / d node| for every node: propagate a unit perturbation."""
    # Rebuild the DAG symbolically with perturbation variables: simplest is to
    # re-trace with node-indexed perturbations in the linear forms.
    n = len(nodes)
    # coefficient of node k's perturbation in each later value: recompute by
    # tracing again with 64 + n dimensional vectors.
    dim = 64 + n
    cnt = [0]

    def rnd(v):
        k = cnt[0]
        cnt[0] += 1
        e = np.zeros(dim)
        e[64 + k] = 1.0
        return v + e

    def aan(d):
        d0, d1, d2, d3, d4, d5, d6, d7 = d
        tmp10 = rnd(d0 + d4); tmp11 = rnd(d0 - d4); tmp13 = rnd(d2 + d6)
        a = rnd(d2 - d6)
        tmp12 = rnd(SQRT2 * a - tmp13)
        e0 = rnd(tmp10 + tmp13); e3 = rnd(tmp10 - tmp13); e1 = rnd(tmp11 + tmp12); e2 = rnd(tmp11 - tmp12)
        z13 = rnd(d5 + d3); z10 = rnd(d5 - d3); z11 = rnd(d1 + d7); z12 = rnd(d1 - d7)
        t7 = rnd(z11 + z13); b = rnd(z11 - z13); t11 = rnd(SQRT2 * b)
        c = rnd(z10 + z12); z5 = rnd(ROT * c)
        t10 = rnd(ROT_P * z12 - z5); t12 = rnd(-ROT_M * z10 + z5)
        t6 = rnd(t12 - t7); t5 = rnd(t11 - t6); t4 = rnd(t10 + t5)
        return [rnd(e0 + t7), rnd(e1 + t6), rnd(e2 + t5), rnd(e3 - t4),
                rnd(e3 + t4), rnd(e2 - t5), rnd(e1 - t6), rnd(e0 - t7)]

    x = [np.eye(dim)[i] for i in range(64)]
    g = [[None] * 8 for _ in range(8)]
    for c in range(8):
        col = aan([x[r * 8 + c] for r in range(8)])
        for r in range(8):
            g[r][c] = col[r]
    outs = []
    for r in range(8):
        outs += aan(g[r])
    outs = np.array(outs)            # (64 outputs, 64 + n)
    return np.abs(outs[:, :64]), np.abs(outs[:, 64:])


def main():
    nodes, out = trace()
    gain, infl = influence(nodes, out)               # (64,64), (64,n)
    mag = np.array([np.abs(v) for v, _ in nodes])    # (n, 64) |dnode/dx|
    cst = np.array([c if c is not None else np.zeros(64) for _, c in nodes])
    K = infl @ mag + infl @ cst + 2.0 * gain          # rounding + constants + inputs
    Kmax = K.max(axis=0)
    # gain bound check: K must dominate the linear gain (used as a range bound)
    assert (Kmax >= gain.max(axis=0)).all()
    lines = ["// GENERATED by tools/analysis/screen_constants.py - do not edit.",
             "// Per-input first-order error weights of the FP32 AAN screen (u = 2^-24 units).",
             "#pragma once",
             "#define HJ_SCREEN_K_INIT { \\"]
    for r in range(8):
        lines.append("  " + ", ".join(f"{float(np.float32(v * 1.0001)):.9g}f" for v in Kmax[r * 8:r * 8 + 8]) + ", \\")
    lines.append("}")
    path = os.path.join(ROOT, "paper_1311_5304_b200", "csrc", "hj_screen.h")
    open(path, "w").write("\n".join(lines) + "\n")
    np.save("/tmp/screen_K.npy", Kmax)
    print("wrote", path, "Kmax range", Kmax.min(), Kmax.max(), "nodes", len(nodes))


if __name__ == "__main__":
    main()
