for sk in 0 2 4 6; do echo "== skip=$sk"; GAPLRA_EPOCH_SKIP=$sk GAPLRA_EPOCH_TIMING=1 timeout 600 python tools/p1_epoch.py C2 20 2>&1 | grep -E "phase" | tail -1; done
