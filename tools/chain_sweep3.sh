run() { echo "== $*"; env "${@:3}" GAPLRA_EPOCH_TIMING=1 timeout 900 python tools/p1_epoch.py $1 $2 2>&1 | grep -E "config|rror" | tail -1 | cut -c90-330; }
run C2 1; run C3 1; run C5 1; run C2 20; run C3 32; run C5 64
run C3 1 GAPLRA_FAST_REDUCER=0 GAPLRA_PUSH_ASYNC=0
run C2 1 GAPLRA_FAST_REDUCER=0 GAPLRA_PUSH_ASYNC=0
