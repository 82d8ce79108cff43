run() { echo "== $1"; shift; env "$@" timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 6 2>&1 | grep -E "rank" ; }
run base GFQ_X=1
run lane0 GFQ_K1_LANE=1
run lane8 GFQ_K1_LANE=1 GFQ_K1_SM_RESERVE=8
run lane16 GFQ_K1_LANE=1 GFQ_K1_SM_RESERVE=16
run lane24 GFQ_K1_LANE=1 GFQ_K1_SM_RESERVE=24
run lane16_green16 GFQ_K1_LANE=1 GFQ_K1_SM_RESERVE=16 GFQ_GREEN_RESERVE=16
run base2 GFQ_X=1
