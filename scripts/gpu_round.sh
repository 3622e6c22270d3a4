#!/bin/bash
# one GPU session: parity tests, then the bench line for every config
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -s -x 2>&1 | grep -E "max\||passed|failed|Error|assert|FAIL" | tail -20
python bench.py --steps 100 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
for c in ${CONFIGS:-c1 c3 c4 c5}; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
