"""Summarise an ncu report (--set full) or a launch-list CSV into text for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep            > profiles/rNN_x.txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv  >> profiles/rNN_x.txt
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = [
    "Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
    "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
    "Theoretical Occupancy", "Dynamic Shared Memory Per Block", "Executed Instructions",
    "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "SM Frequency",
    "Grid Size", "Block Size",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
       "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum"]


def run(args):
    return subprocess.run([NCU, *args], capture_output=True, text=True).stdout


def details(rep):
    out = collections.OrderedDict()
    for row in csv.DictReader(io.StringIO(run(["-i", rep, "--page", "details", "--csv"]))):
        k = row.get("Metric Name", "")
        if k in KEYS and k not in out:
            out[k] = (row.get("Metric Value", ""), row.get("Metric Unit", ""), row.get("Kernel Name", ""))
    return out


def raw(rep):
    rows = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "raw", "--csv"]))))
    if len(rows) < 3:
        return {}
    h, u, v = rows[0], rows[1], rows[2]
    res = {}
    for i, name in enumerate(h):
        if name in RAW or "pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
            res[name] = (v[i], u[i])
    return res


def sass_mix(rep, top=18):
    rows = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "source", "--csv",
                                            "--print-source", "sass"]))))
    if len(rows) < 3:
        return []
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    cnt = collections.Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[idx["Source"]].strip().split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
        cnt[op.split(".")[0]] += int(r[idx["Instructions Executed"]] or 0)
    tot = sum(cnt.values()) or 1
    return [(op, n, n / tot) for op, n in cnt.most_common(top)]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}


def to_bytes(v, u):
    return float(str(v).replace(",", "") or 0) * SCALE.get(u.strip(), 1)


def report(rep):
    d = details(rep)
    name = next(iter(d.values()))[2] if d else "?"
    print(f"# ncu --set full: {rep}\nkernel: {name}\n")
    for k, (v, u, _) in d.items():
        print(f"{k:40s} {v:>16s} {u}")
    r = raw(rep)
    if r:
        print("\n## raw")
        stalls = []
        for k, (v, u) in r.items():
            if "pcsamp" in k:
                stalls.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v))
            else:
                print(f"{k:48s} {v:>16s} {u}")
        rd = to_bytes(*r.get("dram__bytes_read.sum", ("0", "byte")))
        wr = to_bytes(*r.get("dram__bytes_write.sum", ("0", "byte")))
        print(f"{'dram traffic (read+write)':48s} {rd + wr:16.0f} byte")
        if stalls:
            print("\n## warp stall samples")
            for k, v in sorted(stalls, key=lambda x: -float(x[1].replace(',', '') or 0))[:12]:
                print(f"{k:32s} {v}")
    mix = sass_mix(rep)
    if mix:
        print("\n## SASS instruction mix (executed warp instructions)")
        for op, n, f in mix:
            print(f"{op:12s} {n:14d} {f * 100:6.2f}%")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > iv and r[iv]:
            try:
                per[r[ik]].append(to_bytes(r[iv], r[iu]) * 1e9)  # -> ns
            except ValueError:
                pass
    tot = sum(sum(v) for v in per.values()) or 1
    print(f"# launch list (gpu__time_duration.sum, cold-cache, serialised): {path}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:90]:90s} n={len(v):5d} mean={sum(v) / len(v) / 1e3:10.1f} us share={sum(v) / tot * 100:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
