#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from an ncu report (reads `ncu --page source`)."""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ia, isrc, ism, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = sum(int(r[ism] or 0) for r in data)
print(f"total samples {tot}, instructions {len(data)}")
idx = sorted(range(len(data)), key=lambda i: -int(data[i][ism] or 0))[:top]
for i in sorted(idx):
    r = data[i]
    print(f"{i:5d} {int(r[ism]):6d} {100*int(r[ism])/tot:5.1f}%  ex={r[iex]:>8}  {r[isrc].strip()}")
