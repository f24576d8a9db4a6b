"""Aggregate ncu stall samples / executed instructions by CUDA source line
(mixed cuda,sass source page).  usage: ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(lambda: [0, 0, ""])
cur_file = ""
hdr = None
last_line, last_src = "", ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    line, src = r[0], r[1]
    if line:
        last_line, last_src = line, src
    else:
        line, src = last_line, last_src
    try:
        s = int(r[4] or 0)
        e = int(r[7] or 0)
    except ValueError:
        continue
    k = (cur_file, line)
    agg[k][0] += s
    agg[k][1] += e
    if src:
        agg[k][2] = src.strip()[:100]
total = sum(v[0] for v in agg.values()) or 1
print("total samples", total)
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*v[0]/total:5.1f}%  exec={v[1]:9d}  {f}:{l}: {v[2]}")
