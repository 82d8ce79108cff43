cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ext.py tests/test_gpu_chief.py -m gpu -x -q -p no:cacheprovider > gpurun_out/chain_tests.log 2>&1; echo "rc=$?" >> gpurun_out/chain_tests.log
for r in 1 2; do for v in old new; do
if [ $v = old ]; then export GFQ_LIB_PATH=$PWD/tools/exp/old/libgfq.so; else unset GFQ_LIB_PATH; fi
for a in "4096 251" "2048 7" "500 3"; do echo -n "$v $a: " >> gpurun_out/chain_ab.log; python tools/one_ech.py $a 0 --time --reps 10 >> gpurun_out/chain_ab.log 2>&1; done
for c in cfg1 cfg3; do echo -n "$v $c: " >> gpurun_out/chain_ab.log; python tools/one_step.py $c 4 --warm --reps 4 >> gpurun_out/chain_ab.log 2>&1; done
done; done
