run() { echo "== $*"; env "${@:3}" GAPLRA_EPOCH_TIMING=1 timeout 900 python tools/p1_epoch.py $1 $2 2>&1 | grep -E "config|epoch_layout|phase|Error|error" | tail -3; }
run C2 20
run C2 20 GAPLRA_V4_ROWS=128
run C3 32
run C3 32 GAPLRA_V4_ROWS=128
run C3 32 GAPLRA_V4_ROWS=128 GAPLRA_CHAIN_XG=2
