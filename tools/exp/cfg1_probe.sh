cd $GRAFT_REPO_ROOT
python tools/one_step.py cfg1 4 --warm --reps 5 --trace gpurun_out/trace_cfg1.csv > gpurun_out/cfg1_step.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg1_launches.csv python tools/one_step.py cfg1 4 >> gpurun_out/cfg1_step.log 2>&1
