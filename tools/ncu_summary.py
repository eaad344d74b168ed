"""Summarise ncu reports / launch lists into the text kept under profiles/.

usage: python tools/ncu_summary.py full  REPORT.ncu-rep [...]
       python tools/ncu_summary.py launches LAUNCHES.csv
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "warp cycles per issued inst"),
]
STALLS = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:110]}")
        for k, name in KEYS:
            if k in d:
                print(f"   {name:32s} {d[k]:>18s} {u.get(k, '')}")
        st = []
        for k, v in d.items():
            m = STALLS.fullmatch(k)
            if m:
                try:
                    st.append((float(v), m.group(1)))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("   top stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))


def launches(path):
    txt = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(txt))))
    agg = defaultdict(list)
    for r in rows:
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name].append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'mean us':>10s} {'share':>7s}")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:7.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        for p in sys.argv[2:]:
            full(p)
    else:
        launches(sys.argv[2])
