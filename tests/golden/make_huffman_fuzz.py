"""Corrupt-stream fixtures for the host Huffman decoders, from the REFERENCE.

Run in the build container only (needs the reference build in oracle/_ref,
made by oracle/build_ref.sh from /root/reference):

    python tests/golden/make_huffman_fuzz.py

For each base case (committed golden JPEGs, with and without restart
intervals) and each seeded corruption of its entropy-coded bytes (byte
overwritten, byte deleted, 0xFF inserted, marker byte changed, truncation),
the reference's native `decode_mcu_rows` (kernels/_native.pyx:195-305) is
driven one MCU row at a time from a fresh cursor - the reference's own
`entropy.decode_rows` loop (entropy.py:133-155).  Recorded per case: the
int64[8] cursor state after every row, the error class of the first failing
row (or none), and a SHA-256 of the coefficient planes when the loop ends.
tests/test_huffman_fuzz.py replays the same corruptions through this repo's
cursor (hj_decode_mcu_rows) and whole-scan decoder (hj_decode_scan_fast).
Output: tests/golden/huffman_fuzz.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref", "patched"))

from hetjpeg import entropy, errors, parser  # noqa: E402
from hetjpeg.kernels import _native  # noqa: E402

BASES = [  # (golden, y blocks per MCU, MCU height)
    ("t200x130_422_q60_rst13", 2, 8),
    ("t256x256_444_q95_rst7", 1, 8),
    ("t200x130_420_q60_rstrow1", 4, 16),
    ("t333x211_422_q95", 2, 8),
    ("t97x61_444_q100", 1, 8),
]
PER_BASE = 120


def corrupt(span: bytes, rng) -> tuple[bytes, list]:
    """One seeded corruption of the entropy-coded span; returns (bytes, ops)."""
    b = bytearray(span)
    kind = int(rng.integers(0, 6))
    i = int(rng.integers(0, len(b)))
    if kind == 0:
        op = ["set", i, int(rng.integers(0, 256))]
    elif kind == 1:
        op = ["del", i]
    elif kind == 2:
        op = ["ins", i, 0xFF]
    elif kind == 3:
        # retarget a marker / stuffing byte when there is one nearby
        j = b.find(b"\xff", i)
        j = j if j >= 0 and j + 1 < len(b) else i
        op = ["set", min(j + 1, len(b) - 1), int(rng.choice([0x00, 0xD0, 0xD3, 0xD7, 0xD9, 0xC4, 0xFF]))]
    elif kind == 4:
        op = ["trunc", int(rng.integers(1, len(b)))]
    else:
        op = ["set", i, int(b[i] ^ (1 << int(rng.integers(0, 8))))]
    return apply_ops(span, [op]), [op]


def apply_ops(span: bytes, ops) -> bytes:
    b = bytearray(span)
    for op in ops:
        if op[0] == "set":
            b[op[1]] = op[2]
        elif op[0] == "del":
            del b[op[1]]
        elif op[0] == "ins":
            b.insert(op[1], op[2])
        elif op[0] == "trunc":
            del b[op[1]:]
    return bytes(b)


ERR = {errors.BitstreamExhausted: "exhausted", errors.BadCode: "badcode", errors.MarkerInScan: "marker"}


def run_reference(data: bytes, scan, geo, ypm: int, rst: int):
    n_mcu = geo.mcus_per_row * geo.mcu_rows
    y = np.zeros((n_mcu * ypm, 64), np.int16)
    cb = np.zeros((n_mcu, 64), np.int16)
    cr = np.zeros((n_mcu, 64), np.int16)
    st = np.zeros(8, np.int64)
    states, err = [], None
    for row in range(geo.mcu_rows):
        try:
            _native.decode_mcu_rows(data, st, scan, y, cb, cr, row, 1, geo.mcus_per_row, ypm, rst)
        except tuple(ERR) as e:  # state is written back before the raise
            err = [row, ERR[type(e)], str(e)]
            states.append(st.tolist())
            break
        states.append(st.tolist())
    h = hashlib.sha256(y.tobytes() + cb.tobytes() + cr.tobytes()).hexdigest()
    return states, err, h


def main():
    rng = np.random.default_rng(20260417)
    cases = []
    for name, ypm, mh in BASES:
        z = np.load(os.path.join(HERE, name + ".npz"))
        blob = bytes(z["jpeg"])
        if ypm == 4:
            # 4:2:0: the reference parser rejects it; drive its decoder with the
            # header's own tables (the golden's coefficients came this way)
            sys.path.insert(0, REPO)
            from paper_1311_5304_b200 import parser as ours
            p = ours.parse_stream(blob)
        else:
            p = parser.parse_stream(blob)
        packed = entropy._pack_scan_tables(p)
        scan = _native.prepare_scan(*packed)
        sp = p.entropy_span
        span = blob[sp.offset:sp.offset + sp.length]
        w, h = p.width, p.height
        mw = 8 if ypm == 1 else 16
        geo = type("G", (), {"mcus_per_row": -(-w // mw), "mcu_rows": -(-h // mh)})
        for k in range(PER_BASE):
            data, ops = corrupt(span, rng) if k else (span, [])
            states, err, hsh = run_reference(data, scan, geo, ypm, p.restart_interval)
            cases.append({"base": name, "ops": ops, "ypm": ypm, "mcus_per_row": geo.mcus_per_row,
                          "mcu_rows": geo.mcu_rows, "restart_interval": p.restart_interval,
                          "states": states, "error": err, "sha256": hsh})
    out = {"generator": "tests/golden/make_huffman_fuzz.py (reference native decode_mcu_rows, "
                        "oracle/_ref/patched)", "cases": cases}
    with open(os.path.join(HERE, "huffman_fuzz.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    n_err = sum(1 for c in cases if c["error"])
    print(f"{len(cases)} cases, {n_err} with a reference error")


if __name__ == "__main__":
    main()
