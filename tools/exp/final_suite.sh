cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final_tests.log
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k cfg5s > gpurun_out/final_cfg5s.log 2>&1; echo "rc=$?" >> gpurun_out/final_cfg5s.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
