#!/bin/bash
# Static SASS census of the bench's factor kernel for a build variant (CPU only):
#   tools/sasscount.sh NAME "-DX=1 ..."  ->  /tmp/sc/NAME.{cubin,sass,log}
cd "$(dirname "$0")/.." && mkdir -p /tmp/sc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -lineinfo -Xptxas -v $2 \
  -I include -cubin -o /tmp/sc/$1.cubin paper_2311_11833_b200/csrc/psp_kernels.cu > /tmp/sc/$1.log 2>&1 || { tail -20 /tmp/sc/$1.log; exit 1; }
K=${3:-factor_kernel_tmemILb1ELi1ELi2ELb0E}
grep -A2 "Compiling entry function.*$K" /tmp/sc/$1.log | grep -o "Used [0-9]* registers\|[0-9]* bytes stack frame, [0-9]* bytes spill stores, [0-9]* bytes spill loads" | tr '\n' ' '; echo
cuobjdump -sass /tmp/sc/$1.cubin | awk -v k="$K" '/Function :/{on=index($0,k)>0} on' > /tmp/sc/$1.sass
python3 - /tmp/sc/$1.sass <<'PY'
import re, sys
from collections import Counter
c = Counter()
for ln in open(sys.argv[1]):
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
    if m:
        op = m.group(2)
        c[op.split('.')[0] + ('.MOV' if op.startswith('IMAD.MOV') else '')] += 1
print(sum(c.values()), ' '.join(f"{k}:{v}" for k, v in c.most_common(14)))
PY
