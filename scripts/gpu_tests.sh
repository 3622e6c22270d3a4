#!/bin/bash
# parity suite (incl. slow full-size cases) with per-test durations, then the default bench line
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -q -m gpu --timeout 300 ${PYTEST_ARGS:-} -s --durations=15 2>&1 | grep -E "max\||passed|failed|Error|error|assert|FAIL|slowest|s call|worst" | tail -${TAIL:-60} > gpurun_out/gputest.txt
cat gpurun_out/gputest.txt | tail -25
if [ -z "$NO_BENCH" ]; then
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print('c5', round(d['value']), d['roofline']['pass_ms'])"
fi
