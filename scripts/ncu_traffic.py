"""DRAM bytes and executed warp instructions of one pass (one launch of each pass
kernel) from an ncu --set full report -> profiles/ncu_traffic_<cfg>.json (read by
bench.py for roofline.traffic and roofline.issue)."""
import csv
import io
import json
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
outp = sys.argv[3] if len(sys.argv) > 3 else f"profiles/ncu_traffic_{cfg}.json"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
seen, total, per, inst, inst_per = set(), 0.0, {}, 0.0, {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    base = name.split("<")[0]
    if base in seen:
        continue
    seen.add(base)
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        b += float(r[i].replace(",", "")) * scale[units[i]]
    per[name] = b
    total += b
    if "smsp__inst_executed.sum" in hdr:
        n = float(r[hdr.index("smsp__inst_executed.sum")].replace(",", ""))
        inst_per[name] = n
        inst += n
res = {"config": cfg, "report": rep, "dram_bytes_per_pass": total, "per_kernel": per,
       "warp_inst_per_pass": inst, "warp_inst_per_kernel": inst_per,
       "note": "ncu --set full, one launch of each pass kernel (cold L2 between replays)"}
json.dump(res, open(outp, "w"), indent=1)
print(json.dumps(res, indent=1))
