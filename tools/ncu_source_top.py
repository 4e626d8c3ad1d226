"""Top source lines of an ncu report by warp-stall samples (needs -lineinfo and --import-source on).
Usage: python tools/ncu_source_top.py REPORT [N]  -> CSV rows: samples, share, file:line, source text."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if not rows:
    sys.exit("no source page")
hdr = rows[0]
def col(*names):
    for n in names:
        for j, h in enumerate(hdr):
            if h.strip().lower() == n.lower():
                return j
    for n in names:
        for j, h in enumerate(hdr):
            if n.lower() in h.lower():
                return j
    return None
cs = col("Warp Stall Sampling (All Samples)", "Warp Stall Sampling")
cl = col("Line", "#")
cf = col("Source", "Address")
print("# columns:", "|".join(hdr[:12]))
data = []
for r in rows[1:]:
    try:
        v = float(r[cs].replace(",", "")) if cs is not None else 0.0
    except (ValueError, IndexError):
        continue
    data.append((v, r))
tot = sum(v for v, _ in data) or 1.0
for v, r in sorted(data, key=lambda x: -x[0])[:N]:
    line = r[cl] if cl is not None else "?"
    src = (r[cf] if cf is not None else "").strip()[:140]
    print(f"{int(v)},{v / tot:.3f},{line},{src}")
