#!/bin/bash
# A/B env combinations: COMBOS="A=1,B=2 A=0" CONFIGS="c1 c2" (each combo in its own process)
mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c2}; do for combo in ${COMBOS:-none}; do
envs=$(echo "$combo" | tr ',' ' ')
[ "$combo" = "none" ] && envs=""
env $envs timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 3 --no-cpu-baseline --no-e2e --no-prof > gpurun_out/abc.json 2>gpurun_out/abc.err
python -c "
import json; d=json.load(open('gpurun_out/abc.json')); print('$c', '$combo', 'MPix/s=%.0f'%d['value'], 'ms=%.4f'%d['ms_per_step'])" 2>&1 | tail -1
done; done
