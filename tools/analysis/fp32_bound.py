"""Offline analysis for the FP32 fast path:
forward-error constants of the scaled AAN DAG and the fraction of real
blocks the resulting rigorous bound would send to the exact FP64 path."""
import sys
import numpy as np

sys.path.insert(0, '/root/repo')
from oracle import oracle  # noqa

SQRT2, ROT, ROT_P, ROT_M = 1.414213562, 1.847759065, 1.082392200, 2.613125930


def aan_nodes(d):
    """One pass, returning outputs and the list of every rounded node value.
    Mirrors the FP32 kernel's op form: FFMA where the reference has mul+add."""
    d0, d1, d2, d3, d4, d5, d6, d7 = d
    nodes = []
    def n(v): nodes.append(v); return v
    tmp10 = n(d0 + d4); tmp11 = n(d0 - d4); tmp13 = n(d2 + d6)
    a = n(d2 - d6); tmp12 = n(a * SQRT2 - tmp13)        # FFMA: one rounding
    e0 = n(tmp10 + tmp13); e3 = n(tmp10 - tmp13); e1 = n(tmp11 + tmp12); e2 = n(tmp11 - tmp12)
    z13 = n(d5 + d3); z10 = n(d5 - d3); z11 = n(d1 + d7); z12 = n(d1 - d7)
    t7 = n(z11 + z13); b = n(z11 - z13); t11 = n(b * SQRT2)
    c = n(z10 + z12); z5 = n(c * ROT)
    t10 = n(ROT_P * z12 - z5); t12 = n(-ROT_M * z10 + z5)   # FFMA
    t6 = n(t12 - t7); t5 = n(t11 - t6); t4 = n(t10 + t5)
    out = [n(e0 + t7), n(e1 + t6), n(e2 + t5), n(e3 - t4), n(e3 + t4), n(e2 - t5), n(e1 - t6), n(e0 - t7)]
    return out, nodes


def idct2d_linear(x, perturb=None):
    """x: (64, k) linear inputs (k columns of basis vectors or values).
    perturb: (node_index, vector) adds a delta at that node.  Returns
    (outputs (64,k), nodes list)."""
    allnodes = []
    g = [[None] * 8 for _ in range(8)]
    for c in range(8):
        outs, nodes = aan_nodes([x[r * 8 + c] for r in range(8)])
        for r in range(8):
            g[r][c] = outs[r]
        allnodes += nodes
    s = [[None] * 8 for _ in range(8)]
    for r in range(8):
        outs, nodes = aan_nodes(g[r])
        s[r] = outs
        allnodes += nodes
    return np.array([s[r][c] for r in range(8) for c in range(8)]), allnodes


# linear coefficients of every node w.r.t. the 64 inputs: feed identity
E = np.eye(64)
out_lin, nodes_lin = idct2d_linear(list(E))
nodes_lin = [np.abs(v) for v in nodes_lin]           # |dnode/dx_i|, each (64,)
N = len(nodes_lin)
# influence of a unit perturbation at node k on every output: recompute with
# a symbolic perturbation by re-running with an extra input... do it numerically:
# the DAG is linear, so d out / d node_k = out(x with node_k += 1) - out(x).
def run_with_perturb(k):
    cnt = [0]
    import builtins
    def aan_p(d):
        d0, d1, d2, d3, d4, d5, d6, d7 = d
        vals = []
        def n(v):
            if cnt[0] == k:
                v = v + 1.0
            cnt[0] += 1
            return v
        tmp10 = n(d0 + d4); tmp11 = n(d0 - d4); tmp13 = n(d2 + d6)
        a = n(d2 - d6); tmp12 = n(a * SQRT2 - tmp13)
        e0 = n(tmp10 + tmp13); e3 = n(tmp10 - tmp13); e1 = n(tmp11 + tmp12); e2 = n(tmp11 - tmp12)
        z13 = n(d5 + d3); z10 = n(d5 - d3); z11 = n(d1 + d7); z12 = n(d1 - d7)
        t7 = n(z11 + z13); b = n(z11 - z13); t11 = n(b * SQRT2)
        c = n(z10 + z12); z5 = n(c * ROT)
        t10 = n(ROT_P * z12 - z5); t12 = n(-ROT_M * z10 + z5)
        t6 = n(t12 - t7); t5 = n(t11 - t6); t4 = n(t10 + t5)
        return [n(e0 + t7), n(e1 + t6), n(e2 + t5), n(e3 - t4), n(e3 + t4), n(e2 - t5), n(e1 - t6), n(e0 - t7)]
    x = [0.0] * 64
    g = [[None] * 8 for _ in range(8)]
    for cc in range(8):
        outs = aan_p([x[r * 8 + cc] for r in range(8)])
        for r in range(8):
            g[r][cc] = outs[r]
    s = []
    for r in range(8):
        s += aan_p(g[r])
    return np.abs(np.array(s))


infl = np.array([run_with_perturb(k) for k in range(N)])   # (N, 64 outputs)
node_abs = np.array(nodes_lin)                             # (N, 64 inputs)
K = infl.T @ node_abs        # (64 outputs, 64 inputs): sum_v |dout/dv| |dv/dx_i|
Kmax = K.max(axis=0)         # per input weight, max over outputs
print("nodes", N, "K max", K.max(), "Kmax per input (8x8):")
print(np.round(Kmax.reshape(8, 8), 1))
np.save('/tmp/aan_K.npy', K)


def flagged_fraction(width=1920, height=1080, q=90, sub="420", safety=2.5):
    from paper_1311_5304_b200 import entropy, parser
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    blob = synth_jpeg(width, height, q, sub, seed=5)
    p = parser.parse_stream(blob)
    c, _ = entropy.decode_all(p, blob)
    qt = qtable_stack(p)
    pre = np.outer(*(2 * [np.array([1.0] + [np.sqrt(2) * np.cos(k * np.pi / 16) for k in range(1, 8)])])).reshape(64) / 8
    u = 2.0 ** -24
    res = {}
    for name, blocks, qq in (("Y", c.y_blocks, qt[0]), ("Cb", c.cb_blocks, qt[1]), ("Cr", c.cr_blocks, qt[2])):
        x = blocks.astype(np.float64) * qq * pre
        E = safety * u * (np.abs(x) @ Kmax) + 1e-9
        # exact float64 outputs through the oracle core
        n = min(len(blocks), 20000)
        s = np.array([oracle.idct_core_f64(blocks[i].astype(np.int32) * qq, True) for i in range(n)])
        v = s + 128.0
        frac = v + 0.5 - np.floor(v + 0.5)            # distance above the rounding boundary
        near = (np.minimum(frac, 1 - frac) <= E[:n, None]) & (v > -1) & (v < 256)
        fl = near.any(axis=1)
        res[name] = (fl.mean(), np.median(E[:n]), E[:n].max())
    return res


if __name__ == "__main__":
    for q in (75, 90, 95):
        print(q, flagged_fraction(q=q))
