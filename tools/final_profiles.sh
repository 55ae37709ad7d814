#!/bin/bash
# End-of-round ncu captures at HEAD (run under gpurun; outputs under gpurun_out/, summaries copied to profiles/):
#  * one 64-column panel launch of the config-2 subdomain reduce (bk_panel_kernel, 8 x n=4184, 16-CTA clusters),
#  * one 16-RHS pass of the config-4 dataflow block solve (block_solve_dataflow),
#  * the launch list of the config-2 reduce.
# Each program is first run without ncu and must exit 0.
cd "$(dirname "$0")/.."
T=${TAG:-r02zc}
O=gpurun_out
mkdir -p $O
REPS=3 python tools/fem_reduce_probe.py > $O/fem_reduce_$T.log 2>&1 || { echo "fem_reduce_probe failed"; exit 1; }
python tools/solve_probe.py > $O/solve_probe_$T.log 2>&1 || { echo "solve_probe failed"; exit 1; }
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:bk_panel_kernel -s 30 -c 1 -f \
  -o $O/ncu_panel_$T python tools/fem_reduce_probe.py > $O/ncu_panel_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_solve_dataflow -s 1 -c 1 -f \
  -o $O/ncu_solve_flow_$T python tools/solve_probe.py > $O/ncu_solve_flow_$T.log 2>&1
REPS=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_cfg2_reduce_$T.csv python tools/fem_reduce_probe.py > $O/ncu_launches_cfg2_$T.log 2>&1
for r in panel solve_flow; do
  [ -f $O/ncu_${r}_$T.ncu-rep ] && python tools/ncu_summary.py $O/ncu_${r}_$T.ncu-rep > $O/ncu_${r}_${T}_summary.txt 2>&1
done
python tools/ncu_agg.py $O/launches_cfg2_reduce_$T.csv > $O/launches_cfg2_reduce_${T}_summary.txt 2>&1
tail -4 $O/fem_reduce_$T.log $O/solve_probe_$T.log
cat $O/ncu_panel_${T}_summary.txt $O/ncu_solve_flow_${T}_summary.txt
head -16 $O/launches_cfg2_reduce_${T}_summary.txt
