"""Instructions executed and stall samples of one kernel per CUDA source line.

usage: python tools/ncu_lines.py REPORT.ncu-rep CUBIN KERNEL_SUBSTRING [top [SRCDIR]]
Maps ncu's SASS rows (by offset from the kernel's first instruction) to source lines
with `nvdisasm -g` (build with -lineinfo)."""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def line_map(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur_fn, line, m = None, None, {}
    for ln in out.splitlines():
        f = re.match(r"\s*\.text\.(\S+):", ln)
        if f:
            cur_fn = f.group(1)
            continue
        g = re.search(r'//## File "(.*?)", line (\d+)', ln)
        if g:
            line = (g.group(1).split("/")[-1], int(g.group(2)))
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if a and cur_fn and kernel in cur_fn:
            m[int(a.group(1), 16)] = line
    return m


def main():
    rep, cubin, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, data = rows[1], rows[2:]
    iE = h.index("Instructions Executed")
    iS = h.index("Warp Stall Sampling (All Samples)")
    num = lambda x: int(x) if x.isdigit() else 0
    base = min(int(r[0], 16) for r in data)
    m = line_map(cubin, kernel)
    ex, st = defaultdict(int), defaultdict(int)
    for r in data:
        ln = m.get(int(r[0], 16) - base)
        ex[ln] += num(r[iE])
        st[ln] += num(r[iS])
    tE, tS = sum(ex.values()), sum(st.values())
    srcdir = sys.argv[5] if len(sys.argv) > 5 else None
    cache = {}

    def text(ln):
        if not (srcdir and ln):
            return ""
        f, n = ln
        if f not in cache:
            try:
                cache[f] = open(f"{srcdir}/{f}").read().splitlines()
            except OSError:
                cache[f] = []
        return cache[f][n - 1].strip()[:70] if n <= len(cache[f]) else ""

    for ln in sorted(ex, key=lambda k: -st[k])[:top]:
        name = f"{ln[0]}:{ln[1]}" if ln else "?"
        print(f"{name:>24} exec {ex[ln] / tE:6.1%} stall {st[ln] / tS:6.1%}  {text(ln)}")


if __name__ == "__main__":
    main()
