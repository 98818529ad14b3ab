for c in C2 C3 C5; do
  echo "== $c default"; GAPLRA_EPOCH_TIMING=1 python tools/p1_epoch.py $c 2>&1 | grep -E "config|epoch_layout|phase" | tail -3
  for rows in 64 128 256; do
    echo "== $c XG LL rows=$rows"; GAPLRA_EPOCH_TIMING=1 GAPLRA_P1_XG=1 GAPLRA_P1_XG_ROWS=$rows timeout 600 python tools/p1_epoch.py $c 2>&1 | grep -E "config|epoch_layout|phase|Error|error" | tail -3
    echo "== $c LA2 XG LL rows=$rows"; GAPLRA_EPOCH_TIMING=1 GAPLRA_P1_LA2=1 GAPLRA_LA2_XG=1 GAPLRA_LA2_ROWS=$rows timeout 600 python tools/p1_epoch.py $c 2>&1 | grep -E "config|epoch_layout|phase|Error|error" | tail -3
  done
  echo "== $c XG counter rows=128"; GAPLRA_XG_LL=0 GAPLRA_P1_XG=1 timeout 600 python tools/p1_epoch.py $c 2>&1 | grep -E "config|Error" | tail -1
done
