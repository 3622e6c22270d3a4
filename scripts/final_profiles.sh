#!/bin/bash
# End-of-round evidence in ONE gpurun call, keeping gpurun_out/ small (< 64 MiB):
# parity + bench lines for every config, ncu launch lists (c2, c5) and --set full
# captures of the pass kernels (every config) reduced on the box to text/json.
mkdir -p gpurun_out /tmp/ncu
bash scripts/gpu_round.sh > gpurun_out/round_final.txt 2>&1
for c in c1 c2 c3 c4 c5; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prof"
  $CMD > /dev/null 2>&1 || { echo "$c plain run failed"; continue; }
  if [ $c = c2 ] || [ $c = c5 ]; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_$c.csv $CMD > /dev/null 2>&1; echo "$c launches rc=$?"
  fi
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k[abc]_t|k[abc]_i|k2_" -s 6 -c 5 \
    -o /tmp/ncu/full_$c -f $CMD > /dev/null 2>&1; echo "$c full rc=$?"
  python scripts/ncu_summary.py /tmp/ncu/full_$c.ncu-rep > gpurun_out/ncu_full_$c.txt
  python scripts/ncu_traffic.py /tmp/ncu/full_$c.ncu-rep $c gpurun_out/ncu_traffic_$c.json > /dev/null
  python scripts/ncu_lines.py /tmp/ncu/full_$c.ncu-rep ka_tile 30 > gpurun_out/ncu_lines_ka_$c.txt
  python scripts/ncu_lines.py /tmp/ncu/full_$c.ncu-rep kb_tile 30 > gpurun_out/ncu_lines_kb_$c.txt
done
du -sh gpurun_out
