#!/bin/bash
# evidence for profiles/r02: default bench line (c5, with e2e + cpu baseline), c4 line, launch list + ncu of c5
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -2 gpurun_out/bench_default.err
python bench.py --config c4 --steps 20 --warmup 3 > gpurun_out/bench_c4_full.json 2> gpurun_out/bench_c4_full.err; tail -2 gpurun_out/bench_c4_full.err
CFG=c5 UNITS=111820800 LAUNCHES=1 bash scripts/ncu_r2.sh
