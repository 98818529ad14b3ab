# One epoch of every dense chain layout at full size (lockstep parity at the config's d, then 4 epochs of a
# solve with per-class times).  GAPLRA_EPOCH_TIMING=1 adds per-phase cycles per block (and serialises the
# side-stream prep: "standalone" epoch times).
run() { echo "== $*"; env "${@:3}" timeout 900 python tools/p1_epoch.py $1 $2 2>&1 | grep -E "config|epoch_layout|phase|rror" | tail -3; }
run C2 1; run C3 1; run C5 1; run C2 20; run C3 32; run C5 64
