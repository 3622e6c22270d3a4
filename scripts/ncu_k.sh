#!/bin/bash
# ncu --set full of the pass kernels on one bench step (after a clean plain run)
mkdir -p gpurun_out
CFG=${CFG:-c2}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k[123]_fast}" -s ${SKIP:-3} -c ${COUNT:-3} -o gpurun_out/prof_$CFG -f $CMD > gpurun_out/ncu_$CFG.log 2>&1
tail -5 gpurun_out/ncu_$CFG.log
