"""Per-CUDA-source-line instruction and stall shares of one kernel (ncu --print-source cuda,sass)."""
import csv, subprocess, sys, io
rep, kre = sys.argv[1], sys.argv[2]
n_top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        st = float(r[4] or 0); ie = float(r[7] or 0)
    except (ValueError, IndexError):
        continue
    res.append((ie, st, f"{fname}:{r[0]}", r[1][:90]))
ti = sum(x[0] for x in res) or 1; ts = sum(x[1] for x in res) or 1
for ie, st, loc, s in sorted(res, key=lambda x: -x[0])[:n_top]:
    print(f"{ie/ti:6.1%} inst {st/ts:6.1%} stall {loc:28s} {s}")
