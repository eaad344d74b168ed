"""Static SASS instruction count of one kernel per source line (nvdisasm -g): where the
code size goes.  usage: python tools/codemap.py k.cubin <kernel-substring> [top]"""
import collections
import re
import subprocess
import sys

txt = subprocess.run(["nvdisasm", "-g", "-c", sys.argv[1]], capture_output=True, text=True).stdout
lines = txt.split("\n")
start = next(i for i, l in enumerate(lines) if re.match(r"\s*\.section\s+\.text\..*" + re.escape(sys.argv[2]), l))
end = next((j for j in range(start + 1, len(lines)) if re.match(r"\s*\.section\s+\.text\.", lines[j])), len(lines))
cur, cnt = None, collections.Counter()
for l in lines[start:end]:
    m = re.search(r"line (\d+)", l)
    if "//##" in l and m:
        cur = int(m.group(1))
        continue
    if re.search(r"/\*[0-9a-f]{4}\*/", l):
        cnt[cur] += 1
src = open("paper_2311_11833_b200/csrc/psp_kernels.cu").read().split("\n")
tot = sum(cnt.values())
print("total", tot)
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{v:5d} {k}  {src[k - 1].strip()[:90] if k else ''}")
