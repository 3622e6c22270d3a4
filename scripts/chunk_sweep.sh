#!/bin/bash
mkdir -p gpurun_out
for cp in ${CPS:-12 24 48}; do for c in ${CONFIGS:-c2}; do
SGWLS_CHUNK_POS=$cp python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_${c}_${cp}.json 2>gpurun_out/sweep_${c}_${cp}.err
python - <<PY
import json; d=json.load(open("gpurun_out/sweep_${c}_${cp}.json"))
print("$c", "chunk=$cp", "MPix/s=%.0f"%d["value"], {k:round(v["ms_per_step_instrumented"],4) for k,v in d["kernels_instrumented"].items()})
PY
done; done
