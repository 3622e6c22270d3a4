"""Instruction shares of a kernel by source REGION (line ranges of sgwls_tile.cuh /
sgwls_device.cuh) from an ncu report with source: separates the per-position work
(weights, elimination, back substitution, averaging, loads) from the per-thread
fixed overhead (index / geometry / separator set-up, stores)."""
import re, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["python", "scripts/ncu_lines.py", rep, kern, "5000"], capture_output=True, text=True).stdout
src = open('paper_1705_01674_b200/csrc/sgwls_tile.cuh').read().split('\n')
def find(pat):
    for i, l in enumerate(src):
        if pat in l: return i + 1
    raise KeyError(pat)
marks = sorted([(n, find(p)) for n, p in [
    ("tile:helpers(row_fma..)", "struct Rec {"), ("load_chunk_k(eager)", "void load_chunk_k("),
    ("load_chunk_lazy", "struct ChunkInL {"), ("lazy_weights", "struct LazyWeights {"),
    ("load_chunk dispatch", "void load_chunk("), ("Win(elim/shift)", "struct Win {"),
    ("spike_forward", "void chunk_spike_forward_impl("), ("BWin", "struct BWin {"),
    ("enter_block", "void enter_block("), ("reduce_super", "void reduce_super("),
    ("reduce_super_fwd", "void reduce_super_fwd("), ("solve_from_bs", "void solve_from_bs("),
    ("maps_backward", "void maps_backward_column("), ("solve_inner", "void solve_inner("),
    ("k2_tree", "void k2_tree_body("), ("ka_chunk", "void ka_chunk("), ("ka_tile body", "ka_tile(const PassGeom"),
    ("interior_solve", "void chunk_interior_solve("), ("average_shfl", "void average_shfl("),
    ("average_direct", "void average_shfl_direct("), ("covering", "void covering("),
    ("apply_map", "void apply_map("), ("kb_tile body", "kb_tile(const PassGeom")]], key=lambda x: x[1])
tot = {}
for line in out.splitlines():
    m = re.match(r"\s*([\d.]+)% inst\s+([\d.]+)% stall (\S+):(\d+)", line)
    if not m: continue
    ins, stl, f, ln = float(m.group(1)), float(m.group(2)), m.group(3), int(m.group(4))
    if f.startswith('sgwls_tile'):
        name = ([n for n, l in marks if l <= ln] or ["tile:top"])[-1]
    else:
        name = f
    t = tot.setdefault(name, [0, 0]); t[0] += ins; t[1] += stl
for k, (a, b) in sorted(tot.items(), key=lambda kv: -kv[1][0]): print(f"{k:28s} inst {a:5.1f}%  stall {b:5.1f}%")
