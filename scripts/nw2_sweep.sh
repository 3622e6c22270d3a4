#!/bin/bash
# sweep KA tile (SGWLS_KA_WARPS) x KB tile (SGWLS_TILE_WARPS)
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c5}; do for a in ${NWAS:-4 8}; do for b in ${NWBS:-4 8}; do
SGWLS_KA_WARPS=$a SGWLS_TILE_WARPS=$b timeout 300 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e --no-prof > gpurun_out/nw2_${c}_${a}_${b}.json 2>gpurun_out/nw2_${c}_${a}_${b}.err
python -c "
import json; d=json.load(open('gpurun_out/nw2_${c}_${a}_${b}.json')); print('$c', 'KA=$a KB=$b', 'MPix/s=%.0f'%d['value'], 'ms=%.4f'%d['ms_per_step'])" 2>&1 | tail -1
done; done; done
