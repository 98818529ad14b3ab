run() { echo "== $*"; env "${@:3}" GAPLRA_EPOCH_TIMING=1 timeout 900 python tools/p1_epoch.py $1 $2 2>&1 | grep -E "config|phase|Error|error|Assert" | tail -2; }
run C5 64
run C2 20
run C5 1
