#!/bin/bash
# Round-2 closing evidence in one gpurun call (gpurun_out/ stays < 64 MiB):
#   full -m gpu suite, the default bench line (c5, with e2e + CPU baseline), the reference arm,
#   the c4 line, device-only lines of c1-c3, the ncu launch list of the default command and
#   ncu --set full summaries / traffic / per-line / per-region tables of every config.
mkdir -p gpurun_out /tmp/ncu
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -s --durations=8 2>&1 | grep -E "max\||passed|failed|Error|error|assert|FAIL|s call" | tail -40 > gpurun_out/gputest.txt
tail -3 gpurun_out/gputest.txt
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -2 gpurun_out/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c5_reference.json 2> gpurun_out/bench_c5_reference.err
python bench.py --config c4 --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err
for c in c3 c2 c1; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --config c5 --secondary --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_secondary.json 2> gpurun_out/bench_c5_secondary.err
for c in c5 c4 c3 c2 c1; do
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']
print('$c', 'MPix/s=%.0f'%d['value'], 'pass_ms=%.4f'%r['pass_ms'], 'frac=%.3f'%r['frac'], ' '.join('%s=%.3f'%(n,v['ms_per_step_instrumented']) for n,v in d.get('kernels_instrumented',{}).items()))"
done
units() { case $1 in c5) echo 111820800;; c4) echo 167772160;; c3) echo 14647296;; c2) echo 2073600;; c1) echo 783360;; esac; }
for c in c5 c4 c3 c2 c1; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prof"
  $CMD > /dev/null 2>&1 || { echo "$c plain run failed"; continue; }
  if [ $c = c5 ]; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_$c.csv $CMD > /dev/null 2>&1; echo "$c launches rc=$?"
    python scripts/launch_shares.py gpurun_out/launches_$c.csv gpurun_out/launches_$c.json > /dev/null
  fi
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ka_tile|kb_tile|k2_tree" -s 6 -c 3 \
    -o /tmp/ncu/full_$c -f $CMD > /dev/null 2>&1; echo "$c full rc=$?"
  python scripts/ncu_summary.py /tmp/ncu/full_$c.ncu-rep > gpurun_out/ncu_full_$c.txt
  python scripts/ncu_traffic.py /tmp/ncu/full_$c.ncu-rep $c gpurun_out/ncu_traffic_$c.json > /dev/null
  for k in ka_tile kb_tile; do
    python scripts/ncu_lines.py /tmp/ncu/full_$c.ncu-rep $k 40 > gpurun_out/ncu_lines_${k}_$c.txt
    python scripts/sass_mix.py /tmp/ncu/full_$c.ncu-rep $k $(units $c) > gpurun_out/sass_mix_${k}_$c.txt
    python scripts/region_shares.py /tmp/ncu/full_$c.ncu-rep $k > gpurun_out/regions_${k}_$c.txt
  done
  ncu -i /tmp/ncu/full_$c.ncu-rep --page details -k regex:kb_tile 2>/dev/null | grep -E "Throughput|Hit Rate|Issue Slots|Eligible|Issued Warp|No Eligible|Mem Pipes|Registers Per|Theoretical Occ|Achieved Occ" > gpurun_out/ncu_details_kb_$c.txt
done
du -sh gpurun_out
