#!/bin/bash
# A/B an environment knob: VAR=name VALS="a b" CONFIGS="c1 c2"
mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c2 c4}; do for v in ${VALS}; do
env $VAR=$v timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 3 --no-cpu-baseline --no-e2e --no-prof > gpurun_out/ab_${c}_$v.json 2>gpurun_out/ab_${c}_$v.err
python -c "
import json; d=json.load(open('gpurun_out/ab_${c}_$v.json')); print('$c', '$VAR=$v', 'MPix/s=%.0f'%d['value'], 'ms=%.4f'%d['ms_per_step'])" 2>&1 | tail -1
done; done
