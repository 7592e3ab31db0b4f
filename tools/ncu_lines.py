"""Per-source-line instruction / stall shares from an ncu report
(--import-source on, -lineinfo):  python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
data, fname, hdr = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue  # SASS rows carry an address; source rows have "-"
    try:
        n = int(r[hdr.index("Instructions Executed")] or 0)
        w = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    data.append((n, w, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(d[0] for d in data) or 1
ws = sum(d[1] for d in data) or 1
print(f"{'inst%':>6} {'stall%':>6}  line")
key = (lambda d: d[1]) if "--stall" in sys.argv else (lambda d: d[0])
for d in sorted(data, key=key, reverse=True)[:top]:
    print(f"{d[0] / tot * 100:6.2f} {d[1] / ws * 100:6.2f}  {d[2]:22s} {d[3]}")
