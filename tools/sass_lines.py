"""Per-source-line executed instructions and stall share of one kernel in an ncu
report (needs the library built with -lineinfo).  Usage:
python tools/sass_lines.py REPORT LIB KERNEL_MANGLED_SUBSTR TOKENS_PER_UNIT [top]"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, lib, kname, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = dis.split("\n")
cur, on, a2l, fname = None, False, {}, {}
for l in lines:
    if re.match(r"^\s*\.text\.", l) or re.match(r"^\.section\s+\.text\.", l):
        on = kname in l
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and on:
        a2l[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, rows = r[1], r[2:]
ia, sa, ad = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Address")
base = int(rows[0][ad], 16)
ex, st = defaultdict(int), defaultdict(int)
for x in rows:
    ln = a2l.get(int(x[ad], 16) - base)
    ex[ln] += int(x[ia]); st[ln] += int(x[sa])
tot, tst = sum(ex.values()), max(1, sum(st.values()))
srcs = {}
print(f"total {tot}  per unit {tot / units:.1f}")
for ln in sorted(ex, key=lambda k: -ex[k])[:top]:
    text = ""
    if ln:
        f = ln[0]
        if f not in srcs:
            p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1510_06549_b200", "csrc", f)
            srcs[f] = open(p).read().split("\n") if os.path.exists(p) else []
        text = srcs[f][ln[1] - 1].strip()[:78] if srcs[f] else ""
    print(f"{str(ln):28s} {ex[ln] / units:7.1f}  {100 * st[ln] / tst:5.1f}%  {text}")
