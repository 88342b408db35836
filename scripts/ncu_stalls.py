#!/usr/bin/env python
"""Summarise an ncu report's source page: stall reasons over all samples and
the instructions with the most samples.  usage: ncu_stalls.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
S = "Warp Stall Sampling (All Samples)"
tot = {s: sum(int(r[ix[s]] or 0) for r in data) for s in stalls}
all_s = sum(int(r[ix[S]] or 0) for r in data)
print("total samples", all_s)
for s, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {s:28s} {v:9d} {v / max(all_s, 1):.3f}")
ops = {}
for r in data:
    op = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
    ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + int(r[ix[S]] or 0)
print("samples by opcode:", sorted(ops.items(), key=lambda x: -x[1])[:12])
for r in sorted(data, key=lambda r: -int(r[ix[S]] or 0))[:top_n]:
    print(r[0][-5:], r[1][:60], r[ix[S]], {s[6:]: r[ix[s]] for s in stalls if r[ix[s]] not in ("0", "")})
