#!/bin/bash
mkdir -p gpurun_out
for nw in ${NWS:-4 8 16}; do for c in ${CONFIGS:-c2 c5}; do
SGWLS_TILE_WARPS=$nw python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/nw_${c}_${nw}.json 2>/dev/null
python - <<PY
import json; d=json.load(open("gpurun_out/nw_${c}_${nw}.json"))
print("$c", "NW=$nw", "MPix/s=%.0f"%d["value"], "ms=%.4f"%d["ms_per_step"], {k:round(v["ms_per_step_instrumented"],4) for k,v in d["kernels_instrumented"].items()})
PY
done; done
