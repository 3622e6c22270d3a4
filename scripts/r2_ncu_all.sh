#!/bin/bash
# ncu --set full of the pass kernels for c4, c3, c2, c1 (traffic / issue jsons for bench.py, summaries)
CFG=c4 UNITS=167772160 KREGEX="ka_tile|kb_tile|k2_tree" bash scripts/ncu_r2.sh
CFG=c3 UNITS=14647296 bash scripts/ncu_r2.sh
CFG=c2 UNITS=2073600 bash scripts/ncu_r2.sh
CFG=c1 UNITS=783360 bash scripts/ncu_r2.sh
rm -f gpurun_out/full_*.ncu-rep
