#!/bin/bash
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/r02/tl_cfg2a.txt
GFQ_PROF_DUMP=gpurun_out/r02/tl_cfg2a.txt timeout 300 python tools/one_step.py cfg2a 4 --warm --reps 1 --prof
python tools/timeline.py gpurun_out/r02/tl_cfg2a.txt 0.25
timeout 300 python tools/one_step.py cfg2a 4 --warm --reps 1 --trace gpurun_out/r02/trace_cfg2a.csv
GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg2a 4 --warm --reps 10 2>&1 | grep -v " 0.000 ms"
