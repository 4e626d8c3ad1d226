"""Summarise an ncu report (--set full) of one kernel: the numbers DESIGN.md and
bench.py's roofline.traffic quote.  Usage: python tools/ncu_summary.py REPORT [out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__t_bytes.sum": "l1_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct_of_peak",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "launch__grid_size": "grid",
    "smsp__average_warp_latency_per_inst_issued.ratio": "cycles_per_issue",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "second": 1e3}


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if KEYS[h] == "duration":
                    d["duration_ms"] = x * SCALE.get(u, 1.0)
                elif u in SCALE and "byte" in u:
                    d[KEYS[h]] = x * SCALE[u]
                else:
                    d[KEYS[h]] = x
        if "dram_read" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d.get("dram_write", 0.0)
        stalls = {}
        for h, v in zip(hdr, vals):
            # warp-state breakdown: cycles stalled per issued instruction, by reason
            name = None
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                name = h.split("stalled_")[1][:-len(".ratio")]
            elif h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                name = h.split("stalled_")[1][:-len("_per_issue_active.ratio")]
            if name and not name.endswith("_not_issued"):
                try:
                    stalls[name] = float(v.replace(",", ""))
                except ValueError:
                    pass
        if stalls:
            d["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        out.append(d)
    return out


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    print(json.dumps(s, indent=1))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(s[0] if len(s) == 1 else s, f, indent=1)
