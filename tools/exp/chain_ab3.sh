cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ext.py -m gpu -x -q -p no:cacheprovider > gpurun_out/chain_tests.log 2>&1; echo "rc=$?" >> gpurun_out/chain_tests.log
bash tools/exp/chain_ab2.sh
