#!/usr/bin/env python3
"""Summarise an ncu report's source page: stall samples per CUDA source line
(top N) and the stall-reason breakdown. usage: ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr, agg, src = None, None, {}, {}
line = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Line No"].strip():
        line = (cur, int(d["Line No"]))
        src[line] = d["Source"].strip()
        try:
            agg[line] = agg.get(line, 0) + int(d["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print(f"total samples {tot}")
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    print(f"{100 * v / tot:5.1f}%  {f}:{l}  {src[(f, l)][:90]}")
