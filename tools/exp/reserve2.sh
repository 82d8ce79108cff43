run() { echo "== $1"; shift; env "$@" timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 4 2>&1 | grep -E "rank" ; }
run base GFQ_X=1
run lane16 GFQ_K1_LANE=1 GFQ_K1_SM_RESERVE=16
run lane32 GFQ_K1_LANE=1 GFQ_K1_SM_RESERVE=32
run green16 GFQ_GREEN_RESERVE=16
run green32 GFQ_GREEN_RESERVE=32
run waves8 GFQ_K1_MAX_WAVES=8
