cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pdl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_tests.log
for r in 1 2; do for v in old new; do
if [ $v = old ]; then export GFQ_LIB_PATH=$PWD/tools/exp/old/libgfq.so; else unset GFQ_LIB_PATH; fi
echo -n "$v 8192 2: " >> gpurun_out/pdl_ab3.log; python tools/one_ech.py 8192 2 0 --time --reps 3 >> gpurun_out/pdl_ab3.log 2>&1
echo -n "$v cfg5s: " >> gpurun_out/pdl_ab3.log; python tools/one_step.py cfg5s 4 --warm --reps 2 >> gpurun_out/pdl_ab3.log 2>&1
done; done
