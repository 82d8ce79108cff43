cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ext.py -m gpu -x -q -p no:cacheprovider > gpurun_out/chain_tests.log 2>&1; echo "rc=$?" >> gpurun_out/chain_tests.log
bash tools/exp/chain_ab2.sh
GFQ_STEP_DEBUG=20 python tools/one_ech.py 4096 251 0 > gpurun_out/step_dbg_4096.log 2>&1
