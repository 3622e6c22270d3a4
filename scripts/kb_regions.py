import re, subprocess, sys
rep = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof_c2.ncu-rep"
kern = sys.argv[2] if len(sys.argv) > 2 else "kb_tile"
out = subprocess.run(["python", "scripts/ncu_lines.py", rep, kern, "2000"], capture_output=True, text=True).stdout
src = open('paper_1705_01674_b200/csrc/sgwls_tile.cuh').read().split('\n')
def find(pat):
    for i, l in enumerate(src):
        if pat in l: return i + 1
names = [("load_chunk", "void load_chunk("), ("Win", "struct Win {"), ("spike_fwd_impl", "void chunk_spike_forward_impl("),
         ("BWin", "struct BWin {"), ("enter_block", "void enter_block("), ("reduce_super", "void reduce_super("),
         ("solve_inner", "void solve_inner("), ("k2_tree", "k2_tree(const PassGeom"), ("ka", "ka_tile(const PassGeom"),
         ("interior_solve", "void chunk_interior_solve("), ("kb_prologue", "kb_tile(const PassGeom"), ("KB1", "// ---- 1. spike-forward"),
         ("KB2", "// ---- 2. lane-per-band"), ("KB3", "// ---- 3. every chunk"), ("KB4", "// ---- 4. averaging"), ("KB5", "// ---- 5. owned")]
marks = sorted([(n, find(p)) for n, p in names if find(p)], key=lambda x: x[1])
tot = {}
for line in out.splitlines():
    m = re.match(r"\s*([\d.]+)% inst\s+([\d.]+)% stall (\S+):(\d+)", line)
    if not m: continue
    ins, stl, f, ln = float(m.group(1)), float(m.group(2)), m.group(3), int(m.group(4))
    name = [n for n, l in marks if l <= ln][-1] if f.startswith('sgwls_tile') and ln >= marks[0][1] else f
    t = tot.setdefault(name, [0, 0]); t[0] += ins; t[1] += stl
for k, (a, b) in sorted(tot.items(), key=lambda kv: -kv[1][0]): print(f"{k:28s} inst {a:5.1f}%  stall {b:5.1f}%")
