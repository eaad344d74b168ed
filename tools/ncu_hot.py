"""Hot SASS instructions and opcode mix of one kernel in an ncu report.
usage: python tools/ncu_hot.py REPORT.ncu-rep [top]"""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed"); iSrc = h.index("Source")
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[iS]) for r in data); tE = sum(num(r[iE]) for r in data)
print(f"samples {tot}  warp-instructions {tE}")
for r in sorted(data, key=lambda r: -num(r[iS]))[:top]:
    print(f"{r[0][-5:]} {num(r[iS]) / tot:6.1%} {num(r[iE]):>10d}  {r[iSrc][:90]}")
c = Counter()
for r in data:
    toks = r[iSrc].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    c[op.split(".")[0]] += num(r[iE])
print(" ".join(f"{k}:{v / tE:.1%}" for k, v in c.most_common(20)))
