"""Top CUDA source lines of an ncu report by warp-stall samples, with executed warp instructions
(needs -lineinfo and --import-source on).
Usage: python tools/ncu_source_top.py REPORT [N]
Output CSV: stall_samples, share, warp_instructions, share, file:line, source text."""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, data = "?", None, []
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1]) if len(r) > 1 else "?"
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", ""))
        inst = float(r[hdr.index("Instructions Executed")].replace(",", ""))
    except (ValueError, IndexError):
        continue
    data.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:120]))
ts = sum(d[0] for d in data) or 1.0
ti = sum(d[1] for d in data) or 1.0
print("stall_samples,share,warp_instructions,share,line,source")
for s, i, loc, src in sorted(data, key=lambda d: -d[0])[:N]:
    print(f"{int(s)},{s / ts:.3f},{int(i)},{i / ti:.3f},{loc},\"{src}\"")
