"""DC-predictor int16 wrap fixtures, from the REFERENCE.

Run in the build container only (reference build in oracle/_ref):

    python tests/golden/make_dc_wrap.py

The reference accumulates each component's DC predictor in 64 bits and wraps
it to int16 only when storing (kernels/_native.pyx:162-163, `pred[0] +=
diff; out[0] = <short>pred[0]`; fallback.py:379-380 likewise through the
int16 plane).  Real encoders never get there, so the scans are crafted: the
headers (tables, frame) of committed golden JPEGs with a hand-written entropy
segment where every block is one DC difference of category 11 (+-2047,
+-1024, ...) followed by EOB, so predictors run far past +-32767 in both
directions - with and without restart intervals (RSTn resets them).  The
reference's own decode_all produces the expected planes.
Output: tests/golden/dc_wrap.npz (jpeg bytes + y/cb/cr planes per case).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref", "patched"))

from hetjpeg import entropy, parser  # noqa: E402


def canonical_codes(spec):
    """symbol -> (code, length) for a DHT spec (ITU T.81 Annex C)."""
    codes, code, k = {}, 0, 0
    for length in range(1, 17):
        for _ in range(spec.counts[length - 1]):
            codes[spec.symbols[k]] = (code, length)
            code += 1
            k += 1
        code <<= 1
    return codes


class Bits:
    def __init__(self):
        self.acc, self.n, self.out = 0, 0, bytearray()

    def put(self, v, n):
        for i in range(n - 1, -1, -1):
            self.acc = (self.acc << 1) | ((v >> i) & 1)
            self.n += 1
            if self.n == 8:
                self.out.append(self.acc)
                if self.acc == 0xFF:
                    self.out.append(0)
                self.acc, self.n = 0, 0

    def flush(self):
        while self.n:
            self.put(1, 1)  # pad with 1-bits
        return bytes(self.out)


def encode_dc(bits, dc_codes, ac_codes, diff):
    mag = abs(diff)
    t = mag.bit_length()
    c, ln = dc_codes[t]
    bits.put(c, ln)
    if t:
        bits.put(diff if diff > 0 else diff + (1 << t) - 1, t)
    c, ln = ac_codes[0x00]  # EOB
    bits.put(c, ln)


def craft(blob, rst_every, seed):
    p = parser.parse_stream(blob)
    rng = np.random.default_rng(seed)
    specs = {(s.table_class.value, s.table_id): canonical_codes(s) for s in p.huffman_specs}
    comps = p.components
    from hetjpeg.parser import geometry_of
    g = geometry_of(p)
    ypm = g.mcu_width // 8
    n_mcu = g.mcus_per_row * g.mcu_rows
    segs, bits, k = [], Bits(), 0
    for m in range(n_mcu):
        if rst_every and m and m % rst_every == 0:
            segs.append(bits.flush() + bytes([0xFF, 0xD0 + k % 8]))
            bits, k = Bits(), k + 1
        for comp, nblk in ((0, ypm), (1, 1), (2, 1)):
            dc = specs[(0, comps[comp].dc_table_id)]
            ac = specs[(1, comps[comp].ac_table_id)]
            for _ in range(nblk):
                sign = 1 if (m // 23) % 2 == 0 else -1  # long runs up, then down
                diff = sign * int(rng.choice([2047, 2047, 1024, 1500, 0, -3]))
                encode_dc(bits, dc, ac, diff)
    segs.append(bits.flush())
    scan = b"".join(segs)
    sp = p.entropy_span
    head = bytearray(blob[:sp.offset])
    if rst_every:
        # insert a DRI segment before SOS
        sos = head.rfind(b"\xff\xda")
        head[sos:sos] = b"\xff\xdd\x00\x04" + rst_every.to_bytes(2, "big")
    return bytes(head) + scan + b"\xff\xd9"


def main():
    out = {}
    for name, base, rst in (("wrap444", "t64x48_444_q75", 0), ("wrap444_rst", "t64x48_444_q75", 20),
                            ("wrap422", "t333x211_422_q95", 0), ("wrap422_rst", "t200x130_422_q60_rst13", 13)):
        blob = bytes(np.load(os.path.join(HERE, base + ".npz"))["jpeg"])
        crafted = craft(blob, rst, seed=len(out))
        p = parser.parse_stream(crafted)
        c, _ = entropy.decode_all(p, crafted)
        out[name + "_jpeg"] = np.frombuffer(crafted, np.uint8)
        out[name + "_y"], out[name + "_cb"], out[name + "_cr"] = c.y_blocks, c.cb_blocks, c.cr_blocks
        dc = c.y_blocks[:, 0].astype(np.int64)
        print(name, "restart", p.restart_interval, "Y DC range", dc.min(), dc.max())
    np.savez_compressed(os.path.join(HERE, "dc_wrap.npz"), **out)


if __name__ == "__main__":
    main()
