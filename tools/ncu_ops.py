"""Opcode histogram (executed warp instructions) of the kernel in an ncu report, from the
source page's SASS view: python tools/ncu_ops.py REPORT.ncu-rep [n_warps]"""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
i_st = h.index("Warp Stall Sampling (All Samples)")
cnt, stall, tot = collections.Counter(), collections.Counter(), 0
for r in rows[2:]:
    if len(r) <= i_ex:
        continue
    try:
        e = int(r[i_ex])
    except ValueError:
        continue
    src = re.sub(r"^@!?U?P\w+\s+", "", r[i_src].strip())
    op = src.split()[0] if src else "?"
    cnt[op] += e
    tot += e
    try:
        stall[op] += int(r[i_st])
    except ValueError:
        pass
nw = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
st = sum(stall.values()) or 1
print(f"total warp instructions {tot}  per warp {tot / nw:.0f}")
for op, c in cnt.most_common(40):
    print(f"{op:30s} {c / tot * 100:5.1f}%  per-warp {c / nw:9.0f}  stall-samples {stall[op] / st * 100:5.1f}%")
