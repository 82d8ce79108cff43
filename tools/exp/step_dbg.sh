cd $GRAFT_REPO_ROOT
GFQ_STEP_DEBUG=40 python tools/one_ech.py 500 3 0 > gpurun_out/step_dbg_500.log 2>&1
GFQ_STEP_DEBUG=400 python tools/one_ech.py 4096 251 0 > gpurun_out/step_dbg_4096.log 2>&1
