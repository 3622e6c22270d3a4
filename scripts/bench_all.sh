#!/bin/bash
# device-only bench lines of every config (no e2e / CPU legs): MPix/s and pass ms
mkdir -p gpurun_out
for c in ${CONFIGS:-c5 c4 c3 c2 c1}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']
k=' '.join('%s=%.3f'%(n,v['ms_per_step_instrumented']) for n,v in d.get('kernels_instrumented',{}).items())
print('$c', 'MPix/s=%.0f'%d['value'], 'pass_ms=%.4f'%r['pass_ms'], 'frac=%.3f'%r['frac'], k)" 2>&1 | tail -1
done
