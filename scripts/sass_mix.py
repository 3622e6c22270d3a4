"""Dynamic SASS opcode mix of one kernel from an ncu report (source page, SASS view).
usage: sass_mix.py REPORT KERNEL_REGEX [units]   (units: divide counts by this many work items)"""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
ii, it, ist = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
mix = collections.Counter(); tmix = collections.Counter(); smix = collections.Counter()
seq = []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= ii or not r[0].startswith("0x"):
        continue
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    op = op.split(".")[0]
    n = float(r[ii] or 0)
    mix[op] += n; tmix[op] += float(r[it] or 0); smix[op] += float(r[ist] or 0)
    seq.append((r[0], r[1], n, float(r[ist] or 0)))
tot = sum(mix.values()); tt = sum(tmix.values()); ts = sum(smix.values()) or 1
print(f"warp instr {tot:.4g}  thread instr {tt:.4g}" + (f"  thread instr/unit {tt/units:.1f}" if units else ""))
for op, n in mix.most_common(40):
    print(f"{op:10s} {n/tot:6.1%}  thr/unit {tmix[op]/units if units else 0:7.2f}  stall {smix[op]/ts:6.1%}")
if len(sys.argv) > 4:
    with open(sys.argv[4], "w") as f:
        for a, s, n, st in seq:
            f.write(f"{a}\t{n:.0f}\t{st:.0f}\t{s}\n")
