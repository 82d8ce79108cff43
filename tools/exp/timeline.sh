#!/bin/bash
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/r02/tl_cfg5s.txt gpurun_out/r02/tl_cfg4.txt
GFQ_PROF_DUMP=gpurun_out/r02/tl_cfg5s.txt timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 1 --prof
python tools/timeline.py gpurun_out/r02/tl_cfg5s.txt 2
GFQ_PROF_DUMP=gpurun_out/r02/tl_cfg4.txt timeout 300 python tools/one_step.py cfg4 4 --warm --reps 1 --prof
python tools/timeline.py gpurun_out/r02/tl_cfg4.txt 1
bash tools/exp/madlog.sh cfg4 | head -30
