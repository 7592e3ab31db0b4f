"""Instruction / stall share per code region (function name ranges) of an
ncu report: python tools/ncu_regions.py rep.ncu-rep"""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
src = {}
hdr, fname = None, "?"
rows = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    rows.append((fname, int(r[0]), r[1], int(r[hdr.index("Instructions Executed")] or 0),
                 int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
# region = enclosing function in the local copy of the source, or a
# "// ----" section comment inside the kernel body
fn_re = re.compile(r"^\s*(?:__global__|__device__)[^(]*?(\w+)\s*\(")
sec_re = re.compile(r"^\s*// -{4,}\s*(.*?)\s*-*$")
maps = {}
for f in {r[0] for r in rows}:
    local = f
    try:
        lines = open(local).read().splitlines()
    except OSError:
        import os
        local = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                             "paper_1311_5304_b200", "csrc", os.path.basename(f))
        try:
            lines = open(local).read().splitlines()
        except OSError:
            lines = []
    cur, m = "?", {}
    for i, t in enumerate(lines, 1):
        a = fn_re.match(t)
        b = sec_re.match(t)
        if a:
            cur = a.group(1)
        elif b and b.group(1):
            cur = cur.split(" / ")[0] + " / " + b.group(1)[:30]
        m[i] = cur
    maps[f] = m
region_of = {(f, ln): maps[f].get(ln, "?") for f, ln, *_ in rows}
inst = collections.Counter()
stall = collections.Counter()
for f, ln, text, n, w in rows:
    k = region_of[(f, ln)]
    inst[k] += n
    stall[k] += w
T = sum(inst.values()) or 1
W = sum(stall.values()) or 1
for k, v in inst.most_common():
    print(f"{k:28s} inst {v / T * 100:5.1f}%  stall {stall[k] / W * 100:5.1f}%")
