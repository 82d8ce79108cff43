run() { echo "== $1"; shift; env "$@" timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 4 2>&1 | grep -E "rank|green|Error|error" | head -3; }
run base GFQ_X=1
run green16_cd16 GFQ_GREEN_RESERVE=16 GFQ_CRIT_GRID=16
run green24_cd24 GFQ_GREEN_RESERVE=24 GFQ_CRIT_GRID=24
run green32_cd32 GFQ_GREEN_RESERVE=32 GFQ_CRIT_GRID=32
run green48_cd48 GFQ_GREEN_RESERVE=48 GFQ_CRIT_GRID=48
