"""Executed instructions and stall samples of one kernel grouped by code region.

usage: python tools/ncu_regions.py REPORT.ncu-rep CUBIN KERNEL_SUBSTRING REGIONS
REGIONS: name=lo-hi,name=lo-hi,... (source-line ranges of psp_kernels.cu).  Every SASS
instruction is attributed to the region holding its line or its inline call
sites (innermost first); instructions outside every region inherit the last region seen in address order
(inlined helpers sit inside their caller's code)."""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def main():
    rep, cubin, kernel, spec = sys.argv[1:5]
    regions = []
    for part in spec.split(","):
        name, rng = part.split("=")
        lo, hi = rng.split("-")
        regions.append((name, int(lo), int(hi)))

    def region(n):
        for name, lo, hi in regions:
            if lo <= n <= hi:
                return name
        return None

    dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    cur_fn, lines, amap, fresh = None, [], {}, True
    for ln in dis.splitlines():
        f = re.match(r"\s*\.text\.(\S+):", ln)
        if f:
            cur_fn = f.group(1)
            continue
        g = re.search(r'//## File "(.*?)", line (\d+)(?: inlined at "(.*?)", line (\d+))?', ln)
        if g:   # one comment per inlining level, innermost first
            if fresh:
                lines, fresh = [], False
            if g.group(1).endswith("psp_kernels.cu"):
                lines.append(int(g.group(2)))
            if g.group(3) and g.group(3).endswith("psp_kernels.cu"):
                lines.append(int(g.group(4)))
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if a:
            fresh = True
            if cur_fn and kernel in cur_fn:
                amap[int(a.group(1), 16)] = lines
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, data = rows[1], rows[2:]
    iE = h.index("Instructions Executed")
    iS = h.index("Warp Stall Sampling (All Samples)")
    num = lambda x: int(x) if x.isdigit() else 0
    base = min(int(r[0], 16) for r in data)
    ex, st = defaultdict(int), defaultdict(int)
    last = "other"
    for r in sorted(data, key=lambda r: int(r[0], 16)):
        ls = amap.get(int(r[0], 16) - base, [])
        reg = None
        for n in ls:   # innermost line first, then its call site
            reg = reg or region(n)
        if reg is None:
            reg = last
        last = reg
        ex[reg] += num(r[iE])
        st[reg] += num(r[iS])
    tE, tS = sum(ex.values()), sum(st.values())
    for k in sorted(ex, key=lambda k: -ex[k]):
        print(f"{k:>14} exec {ex[k] / tE:6.1%} ({ex[k]:>11d})  stall {st[k] / tS:6.1%}")


if __name__ == "__main__":
    main()
