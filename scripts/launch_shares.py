"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into per-kernel
launch counts, total device time and share; the last whole filter's sequence too.
usage: python scripts/launch_shares.py gpurun_out/launches_c2.csv [out.json]"""
import csv
import io
import json
import re
import sys

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
per = {}
seq = []
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void ", "", r["Kernel Name"]).split("(")[0]
    name = re.sub(r"sgwls_b200::(tile::)?", "", name)
    ns = float(r["Metric Value"].replace(",", ""))
    d = per.setdefault(name, {"launches": 0, "ns": 0.0})
    d["launches"] += 1
    d["ns"] += ns
    seq.append((name, ns, r["Grid Size"], r["Block Size"]))
tot = sum(v["ns"] for v in per.values()) or 1.0
ours = {k: v for k, v in per.items() if not k.startswith(("at::", "elementwise", "vectorized"))}
tot_ours = sum(v["ns"] for v in ours.values()) or 1.0
out = {
    "source": path,
    "note": "ncu --metrics gpu__time_duration.sum --clock-control none: serialised, cold-cache launches; "
            "compare shares, not absolute times",
    "kernels": {k: {"launches": v["launches"], "total_us": v["ns"] / 1e3, "mean_us": v["ns"] / v["launches"] / 1e3,
                    "share_of_library_time": v["ns"] / tot_ours}
                for k, v in sorted(ours.items(), key=lambda kv: -kv[1]["ns"])},
    "other_kernels_us": (tot - tot_ours) / 1e3,
    "launches_listed": len(seq),
}
s = json.dumps(out, indent=1)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(s + "\n")
print(s)
