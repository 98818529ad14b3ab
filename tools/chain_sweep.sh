# p = 1 chains (paired clusters vs one cluster) and the v4 chains after the reducer rewrite
run() { echo "== $*"; env "${@:3}" GAPLRA_EPOCH_TIMING=1 timeout 900 python tools/p1_epoch.py $1 $2 2>&1 | grep -E "config|epoch_layout|phase|Error|error|Assert" | tail -3; }
run C2 1
run C2 1 GAPLRA_P1_PAIR=0
run C5 1
run C5 1 GAPLRA_P1_PAIR=0
run C3 1
run C2 20
run C3 32
run C5 64
