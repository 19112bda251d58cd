"""Split an ncu SASS source page (tools/ncu_capture.sh *_src.csv) into regions
between barriers / branch targets and print executed instructions and stall
samples per region, so the expensive parts of a kernel stand out.
usage: python tools/ncu_regions.py gpurun_out/<tag>_src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ia, isrc, iss, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ins = [(r[ia], r[isrc].strip(), int(r[iss] or 0), int(r[iex] or 0)) for r in rows[2:] if len(r) > iex]
tot_s = sum(x[2] for x in ins) or 1
tot_e = sum(x[3] for x in ins) or 1
# regions: cut at BAR / SYNCS / EXIT
regs, cur = [], []
for x in ins:
    cur.append(x)
    if any(k in x[1] for k in ("BAR.", "SYNCS.PHASECHK", "EXIT", "BRA.U.ANY")):
        regs.append(cur)
        cur = []
if cur:
    regs.append(cur)
out = []
for g in regs:
    s = sum(x[2] for x in g)
    e = sum(x[3] for x in g)
    out.append((s, e, g[0][0][-5:], g[-1][0][-5:], len(g), g[-1][1][:60]))
print(f"total stall samples {tot_s}, executed {tot_e}")
for s, e, a, b, n, last in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% stalls {100*e/tot_e:5.1f}% inst  [{a}..{b}] n={n:4d}  ends: {last}")
