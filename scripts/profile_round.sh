#!/bin/bash
# Profiling evidence for profiles/: launch list (every launch, device time) of the
# default bench command, then one --set full capture of the pass kernels.
# Each ncu runs only after the same command exited 0 without ncu.
mkdir -p gpurun_out
CFG=${CFG:-c2}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prof"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launches_$CFG.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/plain2_$CFG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k[ab2]_t}" -s ${SKIP:-12} -c ${COUNT:-3} \
    -o gpurun_out/full_$CFG -f $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo "full rc=$?"
