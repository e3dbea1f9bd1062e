"""Per-source-line totals (stall samples, warp instructions, L2 sectors) from
`ncu -i rep --page source --csv --print-source=cuda,sass` output.

    python tools/ncu_lines.py dump.csv [top_n]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = None
per = defaultdict(lambda: [0, 0, 0, ""])
hdr = None
line = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        line = (cur_file, int(r[0]), r[1].strip()[:70])
    if not line:
        continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ex = int(r[hdr.index("Instructions Executed")] or 0)
        l2 = r[hdr.index("L2 Theoretical Sectors Global")] if "L2 Theoretical Sectors Global" in hdr else "0"
        l2 = int(l2 or 0) if l2.isdigit() else 0
    except ValueError:
        continue
    k = (line[0], line[1])
    per[k][0] += s
    per[k][1] += ex
    per[k][2] += l2
    per[k][3] = line[2]
tot = sum(v[0] for v in per.values()) or 1
tl2 = sum(v[2] for v in per.values()) or 1
print(f"total samples {tot}, L2 sectors {tl2}")
for k, v in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:5d} {100*v[0]/tot:5.1f}% inst {v[1]:>12d} l2 {100*v[2]/tl2:5.1f}%  {v[3]}")
