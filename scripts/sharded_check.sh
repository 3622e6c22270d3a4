#!/bin/bash
# GPU check of the line-slab sharded path on one device (shards run in one process)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sharded.py -q -m gpu -s -x 2>&1 | grep -E "sharded G|passed|failed|Error|assert" | tail -12
for ls in 1 4; do
timeout 300 python bench.py --config c5 --sharded --local-shards $ls --steps 10 --warmup 3 --no-cpu-baseline --no-prof > gpurun_out/sh_c5_$ls.json 2> gpurun_out/sh_c5_$ls.err; tail -3 gpurun_out/sh_c5_$ls.err
python -c "
import json; d=json.load(open('gpurun_out/sh_c5_$ls.json')); print('c5 local-shards=$ls', round(d['value']), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['gpu_launches'])"
done
