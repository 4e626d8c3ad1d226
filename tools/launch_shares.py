"""Per-kernel mean duration and share of an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X`).
Usage: python tools/launch_shares.py launches.csv [out.txt]"""
import collections
import csv
import sys


def main(path, out=None):
    tot, cnt, unit, hdr = collections.defaultdict(float), collections.Counter(), "", None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                n = d["Kernel Name"]
                tot[n] += float(d["Metric Value"].replace(",", ""))
                cnt[n] += 1
                unit = d["Metric Unit"]
    s = sum(tot.values())
    lines = [f"# {path}: per-kernel mean launch time ({unit}), launches, share of all listed launches "
             f"(ncu: cold-cache, serialised)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{v / cnt[k]:12.1f} x{cnt[k]:4d} share {v / s:.3f}  {k}")
    txt = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(txt)
    print(txt, end="")


if __name__ == "__main__":
    main(*sys.argv[1:])
