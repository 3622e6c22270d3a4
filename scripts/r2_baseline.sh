#!/bin/bash
# round-2 baseline: parity suite, then the default (c5) bench line and c4/c2 lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/gputest.txt
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err
for c in c4 c2 c3 c1; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
cat gpurun_out/gputest.txt
