#!/bin/bash
# A/B library variants: LIBS="default kb3 kb4" CONFIGS="c2 c5"
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c5}; do for v in ${LIBS}; do
if [ "$v" = default ]; then L=paper_1705_01674_b200/libsgwls_b200.so; else L=paper_1705_01674_b200/variants/lib_$v.so; fi
SGWLS_B200_LIB=$L timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 3 --no-cpu-baseline --no-e2e --no-prof > gpurun_out/abl_${c}_$v.json 2>gpurun_out/abl_${c}_$v.err
python -c "
import json; d=json.load(open('gpurun_out/abl_${c}_$v.json')); print('$c', '$v', 'MPix/s=%.0f'%d['value'], 'ms=%.4f'%d['ms_per_step'])" 2>&1 | tail -1
done; done
