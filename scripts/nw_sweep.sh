#!/bin/bash
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c5}; do for nw in ${NWS:-4 8}; do
SGWLS_TILE_WARPS=$nw python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e --no-prof > gpurun_out/nw_${c}_${nw}.json 2>gpurun_out/nw_${c}_${nw}.err
python - <<PY
import json; d=json.load(open("gpurun_out/nw_${c}_${nw}.json"))
print("$c", "NW=$nw", "MPix/s=%.0f"%d["value"], "ms=%.4f"%d["ms_per_step"], "frac=%.3f"%d["roofline"]["frac"])
PY
done; done
