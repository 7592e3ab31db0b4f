"""Generate the pinned float64 constant tables as C headers.

Restates the table formulas of the reference (`pkg/src/hetjpeg/kernels/
constants.py:9-49`) with numpy and writes them as hex-float literals, so the
CUDA kernels and the CPU oracle use bit-identical constants without calling
`cos` on the device.  When the reference package is importable (the build
container), every value is asserted bit-equal to the reference's own arrays.

Outputs:
  paper_1311_5304_b200/csrc/hj_tables.h   (product)
  oracle/oracle_tables.h                  (test oracle; same numbers)
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def tables():
    # constants.py:9-19 - zigzag position k -> natural index
    zz = []
    for s in range(15):  # anti-diagonals r + c = s
        rows = list(range(max(0, s - 7), min(s, 7) + 1))
        if s % 2 == 0:   # even diagonals run bottom-left -> top-right
            rows.reverse()
        zz.extend(r * 8 + (s - r) for r in rows)
    zz = np.array(zz, dtype=np.int32)
    # constants.py:21-29 - separable basis 0.5*C_u*cos((2x+1)u*pi/16)
    u = np.arange(8).reshape(8, 1).astype(np.float64)
    x = np.arange(8).reshape(1, 8).astype(np.float64)
    basis = 0.5 * np.cos((2.0 * x + 1.0) * u * np.pi / 16.0)
    basis[0, :] *= 1.0 / np.sqrt(2.0)
    # constants.py:31-35 - decimal rotator literals
    rot = {"SQRT2": 1.414213562, "ROT": 1.847759065, "ROT_P": 1.082392200,
           "ROT_M": 2.613125930}
    # constants.py:37-43 - prescale outer(s, s) / 8
    s = np.empty(8, dtype=np.float64)
    s[0] = 1.0
    for k in range(1, 8):
        s[k] = np.sqrt(2.0) * np.cos(k * np.pi / 16.0)
    pre = np.outer(s, s) / 8.0
    # constants.py:45-49 - colour weights
    colour = {"CR_TO_R": 1.402, "CB_TO_G": 0.34414, "CR_TO_G": 0.71414,
              "CB_TO_B": 1.772}
    return zz, basis, rot, pre, colour


COLOR_K = 20


def colour_constants():
    """Integer formulas equal to the reference's float64 colour rounding.

    The reference computes R = round_u8(Y + 1.402(Cr-128)) etc. in float64
    (_native.pyx:391-395, fallback.py:142-150).  Searched here and verified
    over all 2^24 (Y, Cb, Cr): R = clamp((Y<<K + AR*Cr + CR) >> K),
    B = clamp((Y<<K + AB*Cb + CB) >> K), G = clamp((Y<<K + AGB*Cb + AGR*Cr
    + CG) >> K) except the single float64 tie pair (Cb, Cr) = (78, 178), whose
    offset is -19 for 47 <= Y <= 82 and -18 otherwise.
    """
    K = COLOR_K
    v = np.arange(256, dtype=np.float64)
    iv = np.arange(256, dtype=np.int64)
    Y = v[:, None, None]
    cb = v[None, :, None]
    cr = v[None, None, :]
    fr = lambda x: np.floor(x + 0.5)  # noqa: E731  (clamp is applied after)
    offR = (fr(200.0 + 1.402 * (v - 128.0)) - 200.0).astype(np.int64)
    offB = (fr(200.0 + 1.772 * (v - 128.0)) - 200.0).astype(np.int64)
    g_all = fr(Y - 0.34414 * (cb - 128.0) - 0.71414 * (cr - 128.0)) - Y
    offG = g_all[200].astype(np.int64)

    def fit1(off, w):
        base = int(round(w * 2 ** K))
        for dA in range(0, 65):
            for A in (base + dA, base - dA):
                lo = (off * 2 ** K - A * iv).max()
                hi = ((off + 1) * 2 ** K - A * iv - 1).min()
                if lo <= hi:
                    return A, int((lo + hi) // 2)
        raise RuntimeError("no fit")

    def fit2(off, wb, wr):
        bb, br = int(round(-wb * 2 ** K)), int(round(-wr * 2 ** K))
        CB, CR = iv[:, None], iv[None, :]
        for dA in range(-40, 41):
            for dB in range(-40, 41):
                s = (bb + dA) * CB + (br + dB) * CR
                lo = (off * 2 ** K - s).max()
                hi = ((off + 1) * 2 ** K - s - 1).min()
                if lo <= hi:
                    return bb + dA, br + dB, int((lo + hi) // 2)
        raise RuntimeError("no fit")

    AR, CR_ = fit1(offR, 1.402)
    AB, CB_ = fit1(offB, 1.772)
    AGB, AGR, CG = fit2(offG, 0.34414, 0.71414)
    # exhaustive verification against the float64 formula over all 2^24 inputs
    yi = np.arange(256, dtype=np.int64)[:, None, None]
    cbi = iv[None, :, None]
    cri = iv[None, None, :]
    clamp = lambda a: np.clip(a, 0, 255)  # noqa: E731
    r_ref = clamp(fr(Y + 1.402 * (cr - 128.0))).astype(np.int64)
    b_ref = clamp(fr(Y + 1.772 * (cb - 128.0))).astype(np.int64)
    g_ref = clamp(fr(Y - 0.34414 * (cb - 128.0) - 0.71414 * (cr - 128.0))).astype(np.int64)
    r_int = clamp(((yi << K) + AR * cri + CR_) >> K)
    b_int = clamp(((yi << K) + AB * cbi + CB_) >> K)
    g_int = ((yi << K) + AGB * cbi + AGR * cri + CG) >> K
    special = (cbi == 78) & (cri == 178) & (yi >= 47) & (yi <= 82)
    g_int = clamp(g_int - special)
    assert np.array_equal(np.broadcast_to(r_int, r_ref.shape), r_ref), "R formula"
    assert np.array_equal(np.broadcast_to(b_int, b_ref.shape), b_ref), "B formula"
    assert np.array_equal(g_int, g_ref), "G formula"
    # the tie pair's G accumulator value must be unique over all (Cb, Cr)
    gsum = AGB * iv[:, None] + AGR * iv[None, :] + CG
    assert (gsum == AGB * 78 + AGR * 178 + CG).sum() == 1, "G special value not unique"
    return {"K": K, "AR": AR, "CR": CR_, "AB": AB, "CB": CB_, "AGB": AGB, "AGR": AGR,
            "CG": CG}


def check_against_reference(zz, basis, rot, pre, colour) -> bool:
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        return False
    sys.path.insert(0, ref)
    os.environ.setdefault("HETJPEG_BACKEND", "fallback")
    from hetjpeg.kernels import constants as C  # noqa: E402
    assert np.array_equal(zz, C.ZIGZAG), "zigzag mismatch"
    assert np.array_equal(basis.view(np.uint64), C.IDCT_BASIS.view(np.uint64)), "basis bits"
    assert np.array_equal(pre.view(np.uint64), C.AAN_PRESCALE.view(np.uint64)), "prescale bits"
    for k, v in rot.items():
        assert float(getattr(C, "AAN_" + k)).hex() == v.hex(), k
    for k, v in colour.items():
        assert float(getattr(C, k)).hex() == v.hex(), k
    return True


def emit(path: str, prefix: str, zz, basis, rot, pre, colour, pinned: bool,
         icol=None) -> None:
    lines = [
        "// GENERATED by tools/gen_constants.py - do not edit.",
        "// Bit-exact float64 tables of the reference (pkg/src/hetjpeg/kernels/constants.py:9-49).",
        f"// Checked bit-equal against the reference module at generation time: {pinned}.",
        "#pragma once",
        "",
        f"#define {prefix}SQRT2 {rot['SQRT2'].hex()}",
        f"#define {prefix}ROT {rot['ROT'].hex()}",
        f"#define {prefix}ROT_P {rot['ROT_P'].hex()}",
        f"#define {prefix}ROT_M {rot['ROT_M'].hex()}",
    ]
    for k, v in colour.items():
        lines.append(f"#define {prefix}{k} {v.hex()}")
    lines.append("")
    lines.append(f"#define {prefix}ZIGZAG_INIT {{ " + ", ".join(str(int(v)) for v in zz) + " }")
    lines.append(f"#define {prefix}PRESCALE_INIT {{ \\")
    for r in range(8):
        lines.append("  " + ", ".join(float(v).hex() for v in pre[r]) + ", \\")
    lines.append("}")
    lines.append(f"#define {prefix}BASIS_INIT {{ \\")
    for r in range(8):
        lines.append("  " + ", ".join(float(v).hex() for v in basis[r]) + ", \\")
    lines.append("}")
    if icol is not None:
        lines.append("")
        lines.append("// integer colour formulas, exhaustively verified over 2^24 inputs")
        for k, v in icol.items():
            lines.append(f"#define {prefix}COL_{k} ({v})")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines) + "\n")


def main() -> None:
    zz, basis, rot, pre, colour = tables()
    pinned = check_against_reference(zz, basis, rot, pre, colour)
    icol = colour_constants()
    emit(os.path.join(ROOT, "paper_1311_5304_b200", "csrc", "hj_tables.h"), "HJ_",
         zz, basis, rot, pre, colour, pinned, icol)
    emit(os.path.join(ROOT, "oracle", "oracle_tables.h"), "OR_",
         zz, basis, rot, pre, colour, pinned)
    print("constants written; reference check:", "passed" if pinned else "skipped")


if __name__ == "__main__":
    main()
