#!/usr/bin/env python
"""Warp-stall samples of an ncu report by CUDA source line (needs -lineinfo and
--import-source on): top lines with their dominant stall reasons.
usage: ncu_lines.py report.ncu-rep [top] [file-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
S = "Warp Stall Sampling (All Samples)"
rows, fname, hdr = [], "", None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and S in hdr and len(r) > hdr[S] and r[0].isdigit() and r[2] == "-" and r[hdr[S]] not in ("", "0"):
        rows.append((fname.split("/")[-1], r, hdr))
tot = sum(int(r[h[S]]) for _, r, h in rows)
print("total samples", tot)
for f, r, h in sorted(rows, key=lambda x: -int(x[1][x[2][S]]))[:top_n]:
    if want and want not in f:
        continue
    st = {k[6:]: int(r[i]) for k, i in h.items() if k.startswith("stall_") and "Not Issued" not in k and r[i] not in ("", "0")}
    st = dict(sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{f}:{r[0]:>5} {int(r[h[S]]) / tot:6.3f}  {r[1].strip()[:70]:70s} {st}")
