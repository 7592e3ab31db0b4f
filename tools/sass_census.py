"""SASS instruction census of the render kernels (static counts per opcode,
and the Blackwell-specific opcodes that prove the code path), from the built
library:   python tools/sass_census.py > profiles/rNN_sass_census.txt"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1311_5304_b200/libhetjpeg_b200.so"
out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
print(f"# cuobjdump -sass {LIB}: static instruction counts per render kernel")
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if "render_kernel" not in name and "render_tc_kernel" not in name and "unpack_blocks" not in name:
        continue
    ops = collections.Counter()
    for line in f.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            ops[m.group(1) + (m.group(2) or "")] += 1
    base = collections.Counter()
    for k, v in ops.items():
        base[k.split(".")[0]] += v
    sub = re.search(r"render_kernelILi(\d)ELi(\d)E", name)
    tcs = re.search(r"render_tc_kernelILi(\d)E", name)
    label = (f"render_kernel<{sub.group(1)},{sub.group(2)}>" if sub else
             f"render_tc_kernel<{tcs.group(1)}>" if tcs else
             "unpack_blocks_kernel" if "unpack_blocks" in name else name)
    print(f"\n## {label}  ({sum(ops.values())} instructions)")
    print("  top opcodes: " + ", ".join(f"{k} {v}" for k, v in base.most_common(24)))
    special = {k: v for k, v in ops.items() if k.split(".")[0] in
               ("FADD2", "FFMA2", "FMUL2", "I2IP", "UBLKPF", "LDG", "LDTM", "UTCBAR", "SYNCS")
               or k.startswith("UTC") or k.startswith("LDG.E.NA") or "256" in k}
    print("  Blackwell / path markers: " + ", ".join(f"{k} {v}" for k, v in sorted(special.items())))
