cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pdl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_tests.log
for r in 1 2; do for v in old new; do
if [ $v = old ]; then export GFQ_LIB_PATH=$PWD/tools/exp/old/libgfq.so; else unset GFQ_LIB_PATH; fi
for c in cfg2a cfg1 cfg3; do echo -n "$v $c: " >> gpurun_out/pdl_ab.log; python tools/one_step.py $c 4 --warm --reps 5 >> gpurun_out/pdl_ab.log 2>&1; done
done; done
