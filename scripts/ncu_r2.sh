#!/bin/bash
# ncu evidence for one config (each ncu run only after the same command exited 0 without ncu):
# launch list of the timed bench command, then --set full + source of the pass kernels,
# reduced on the box to text (summary, per-line hot spots, dynamic SASS opcode mix).
mkdir -p gpurun_out
CFG=${CFG:-c5}
UNITS=${UNITS:-0}   # band positions per pass (per-unit instruction counts)
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prof"
$CMD > gpurun_out/plain_$CFG.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$CFG.log; exit 1; }
if [ -n "$LAUNCHES" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$CFG.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
fi
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-ka_tile|kb_tile|k2_tree}" \
  -s ${SKIP:-6} -c ${COUNT:-3} -o /tmp/full_$CFG -f $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo "full rc=$?"
python scripts/ncu_summary.py /tmp/full_$CFG.ncu-rep > gpurun_out/ncu_full_$CFG.txt
for k in ka_tile kb_tile; do
  python scripts/ncu_lines.py /tmp/full_$CFG.ncu-rep $k 40 > gpurun_out/ncu_lines_${k}_$CFG.txt
  python scripts/sass_mix.py /tmp/full_$CFG.ncu-rep $k $UNITS > gpurun_out/mix_${k}_$CFG.txt
done
python scripts/ncu_traffic.py /tmp/full_$CFG.ncu-rep $CFG gpurun_out/ncu_traffic_$CFG.json > /dev/null 2>&1
cp /tmp/full_$CFG.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
