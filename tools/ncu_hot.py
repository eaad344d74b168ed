"""Hot SASS instructions, opcode mix and stall reasons of one kernel in an ncu report.

usage: python tools/ncu_hot.py REPORT.ncu-rep [top]          hot instructions + opcode mix
       python tools/ncu_hot.py --stalls REPORT.ncu-rep [top] stall reasons per instruction
       python tools/ncu_hot.py --buckets REPORT.ncu-rep UNITS instructions by execution count
"""
import csv
import subprocess
import sys
from collections import Counter, defaultdict


def _rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[1], rows[2:]


def _num(x):
    return int(x) if x.isdigit() else 0


def hot(rep, top=30):
    h, data = _rows(rep)
    iS = h.index("Warp Stall Sampling (All Samples)")
    iE = h.index("Instructions Executed")
    iSrc = h.index("Source")
    tot = sum(_num(r[iS]) for r in data)
    tE = sum(_num(r[iE]) for r in data)
    print(f"samples {tot}  warp-instructions {tE}")
    for r in sorted(data, key=lambda r: -_num(r[iS]))[:top]:
        print(f"{r[0][-5:]} {_num(r[iS]) / tot:6.1%} {_num(r[iE]):>10d}  {r[iSrc][:90]}")
    c = Counter()
    for r in data:
        toks = r[iSrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        c[op.split(".")[0]] += _num(r[iE])
    print(" ".join(f"{k}:{v / tE:.1%}" for k, v in c.most_common(20)))


def stalls(rep, top=30):
    h, data = _rows(rep)
    iSrc = h.index("Source")
    iW = h.index("Warp Stall Sampling (All Samples)")
    sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(_num(r[iW]) for r in data)
    agg = defaultdict(int)
    for r in data:
        for i in sc:
            agg[h[i][6:]] += _num(r[i])
    print("stall totals:", ", ".join(f"{k}={v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:9]))
    for r in sorted(data, key=lambda r: -_num(r[iW]))[:top]:
        reasons = sorted(((_num(r[i]), h[i][6:]) for i in sc), reverse=True)[:2]
        print(f"{r[0][-5:]} {_num(r[iW]) / tot:5.1%} {r[iSrc][:62]:62s} " +
              " ".join(f"{n}:{v}" for v, n in reasons if v))


def buckets(rep, units):
    h, data = _rows(rep)
    iE = h.index("Instructions Executed")
    iW = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(_num(r[iE]) for r in data)
    ts = sum(_num(r[iW]) for r in data)
    b, nb, st = defaultdict(int), defaultdict(int), defaultdict(int)
    for r in data:
        e = _num(r[iE])
        k = round(e / units)
        b[k] += e
        nb[k] += 1
        st[k] += _num(r[iW])
    print(f"instructions per unit {tot / units:.0f}")
    for k in sorted(b, key=lambda k: -b[k])[:20]:
        print(f"exec/unit {k:8d}  instrs {nb[k]:5d}  share {b[k] / tot:6.1%}  per-unit {b[k] / units:9.0f}"
              f"  stall-samples {st[k] / ts:6.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "--stalls":
        stalls(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
    elif sys.argv[1] == "--buckets":
        buckets(sys.argv[2], float(sys.argv[3]))
    else:
        hot(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
