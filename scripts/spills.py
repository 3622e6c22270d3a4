"""ptxas register / spill table of the tile kernels: python scripts/spills.py [extra nvcc flags]"""
import re, subprocess, sys
flags = sys.argv[1:]
for r in (1, 2, 3, 4):
    out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
                          "-Iinclude", "-Xptxas", "-v", "-c", f"paper_1705_01674_b200/csrc/tile_r{r}.cu", "-o", "/tmp/t.o"] + flags,
                         capture_output=True, text=True).stderr
    cur = None
    for line in out.splitlines():
        m = re.search(r"Compiling entry function '_ZN10sgwls_b2004tile(\d+)(\w+?)ILi(\d)ELi(\d)(?:ELi(\d))?", line)
        if m:
            cur = f"{m.group(2)}<{m.group(3)},{m.group(4)}" + (f",{m.group(5)}>" if m.group(5) else ">")
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            sp = (int(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and cur.startswith(("ka_tile", "kb_tile", "k2_tree")):
            print(f"{cur:18s} regs {m.group(1):>3s}  spill st/ld {sp[0]:5d} {sp[1]:5d}")
            cur = None
