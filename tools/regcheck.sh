#!/bin/bash
# Compile psp_kernels.cu alone (sm_100a) and report registers / stack / spills of the
# factor and solve kernels (ptxas -v) — a quick check before a GPU run.
set -e
cd "$(dirname "$0")/.."
out=${1:-/tmp/regcheck}
mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -lineinfo -Xptxas -v \
  -I include -cubin -o $out/k.cubin paper_2311_11833_b200/csrc/psp_kernels.cu > $out/ptxas.log 2>&1
python3 - "$out/ptxas.log" <<'PY'
import re, sys
name = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name and ('tmem' in name or 'solve' in name):
        st = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and name and ('tmem' in name or 'solve_kernel' in name):
        print(f"{name[-48:]:50s} regs {m.group(1)} stack/spill {st}")
        name = None
PY
