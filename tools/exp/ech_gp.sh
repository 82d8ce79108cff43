#!/bin/bash
# general-p ECH: wall time and launch lists of one 4096^2 GF(251) and one
# 2048^2 GF(7) block (the cfg4 / cfg3 diagonal blocks)
mkdir -p gpurun_out
for a in "4096 251" "2048 7" "8192 251"; do
  set -- $a
  timeout 120 python tools/one_ech.py $1 $2 0 --time --reps 5 > gpurun_out/echgp_time_$1_$2.log 2>&1
  GFQ_STEP_DEBUG=200 timeout 120 python tools/one_ech.py $1 $2 0 > gpurun_out/echgp_dbg_$1_$2.log 2>&1
done
for a in "4096 251" "2048 7"; do
  set -- $a
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/echgp_launch_$1_$2.csv python tools/one_ech.py $1 $2 0 > /dev/null 2>&1
done
