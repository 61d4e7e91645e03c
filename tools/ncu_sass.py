#!/usr/bin/env python
"""SASS of the hottest region with execution counts: python tools/ncu_sass.py REP [min_count] [file:line-range]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; mn = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
rng = None
if len(sys.argv) > 3:
    f, r = sys.argv[3].split(":"); a, b = map(int, r.split("-")); rng = (f, a, b)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname = None; hdr = None; cur = None
for r in csv.reader(io.StringIO(src)):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]
    if len(r) > 5 and r[0] == "Line No": hdr = r; continue
    if not hdr or len(r) < 8: continue
    if r[0] != "" and r[2] == "-": cur = (fname, int(r[0])); continue
    if r[0] == "" and r[7] not in ("-", "") and float(r[7]) >= mn:
        if rng and not (cur[0] == rng[0] and rng[1] <= cur[1] <= rng[2]): continue
        print(f"{cur[0]}:{cur[1]:<5d} {r[2][-5:]} {int(r[7]):>10d}  {r[3].strip()[:90]}")
