cd $GRAFT_REPO_ROOT
GFQ_HOSTPROF=1 python tools/one_step.py cfg5s 4 --warm --reps 4 > gpurun_out/cfg5_var.log 2>&1
