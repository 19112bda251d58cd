"""Summarise an ncu capture exported by tools/ncu_capture.sh (raw + source
CSV pages): key metrics, stall reasons, opcode mix.  usage:
    python tools/ncu_summary.py gpurun_out/<tag>  "<header line>" > profiles/<name>.txt"""
import collections
import csv
import re
import sys

base, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = list(csv.reader(open(base + "_raw.csv")))
h, u = rows[0], rows[1]
KEYS = ("Kernel Name|gpu__time_duration.sum$|dram__bytes_read.sum$|dram__bytes_write.sum$|"
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|launch__registers_per_thread$|"
        "launch__grid_size|launch__block_size|sm__warps_active.avg.pct_of_peak_sustained_active|"
        "smsp__issue_active.avg.pct_of_peak_sustained_active|sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|"
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active|lts__t_sector_hit_rate.pct$|"
        "l1tex__m_xbar2l1tex_read_bytes.sum$|lts__throughput.avg.pct_of_peak_sustained_elapsed|smsp__inst_executed.sum$")
print("#", header)
for r in rows[2:]:
    for k, unit, v in zip(h, u, r):
        if re.search(KEYS, k) and not k.startswith(("LTS.", "SM_A.", "TPC.")):
            print(f"{k:72s} {v[:100]} {unit}")
    stalls = [(k, v) for k, v in zip(h, r) if re.search(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active", k)]
    stalls = sorted(((float(v or 0), re.search(r"stalled_(\w+)_per", k).group(1)) for k, v in stalls), reverse=True)
    print("# stall reasons (warps per issue, top 8): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))
src = list(csv.reader(open(base + "_src.csv")))
hh = src[1]
i_src, i_e = hh.index("Source"), hh.index("Instructions Executed")
op = collections.Counter()
for r in src[2:]:
    if len(r) > i_e and r[i_e]:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[i_src].strip())
        if m:
            op[m.group(2)] += int(r[i_e])
tot = sum(op.values())
print("# opcode mix (warp-level executed): " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in op.most_common(10)))
