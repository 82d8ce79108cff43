cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in old new; do
case $v in old) export GFQ_LIB_PATH=$PWD/tools/exp/old/libgfq.so;; c) export GFQ_LIB_PATH=$PWD/tools/exp/c/libgfq.so;; *) unset GFQ_LIB_PATH;; esac
for a in "4096 251" "2048 7" "500 3"; do echo -n "$v $a: " >> gpurun_out/chain_ab.log; python tools/one_ech.py $a 0 --time --reps 10 >> gpurun_out/chain_ab.log 2>&1; done
echo -n "$v cfg1: " >> gpurun_out/chain_ab.log; python tools/one_step.py cfg1 4 --warm --reps 5 >> gpurun_out/chain_ab.log 2>&1
done; done
