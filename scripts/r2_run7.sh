#!/bin/bash
NO_BENCH=1 TEST_TIMEOUT=600 bash scripts/gpu_tests.sh
STEPS=30 bash scripts/bench_all.sh
timeout 600 python scripts/multi_local.py 2 4 8 > gpurun_out/multi_local.txt 2>&1; tail -5 gpurun_out/multi_local.txt
timeout 300 python bench.py --config c5 --sharded --shard-mode slabs --local-shards 8 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sh_slabs8.json 2> gpurun_out/sh_slabs8.err; tail -2 gpurun_out/sh_slabs8.err
timeout 600 python bench.py --config c5 --sharded --shard-mode transpose --local-shards 8 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sh_transpose8.json 2> gpurun_out/sh_transpose8.err; tail -2 gpurun_out/sh_transpose8.err
python -c "
import json
for f in ['sh_slabs8','sh_transpose8']:
    try:
        d=json.load(open('gpurun_out/%s.json'%f)); print(f, round(d['value']), d['ms_per_step'], {k:round(v['ms_per_step_instrumented'],3) for k,v in d['kernels_instrumented'].items()})
    except Exception as e: print(f, e)
"
