#!/bin/bash
# build + time the ws kernel for several G unit sizes (positions per G unit)
for gp in ${GPS:-1 2 4}; do
  touch paper_1912_02165_b200/csrc/fused_ws.cu; make -s -j8 EXTRA="-DWF_WS_GP=$gp" >/dev/null 2>&1 || { echo "build gp=$gp failed"; continue; }
  for l in ${LAGS:-24 32 48}; do
    echo "gp $gp lag $l: $(timeout 60 python tools/ws_time.py c2 10 WF_WS_LAG=$l WF_WS_BUDGET_MB=${BUDGET:-300} | grep -v "WF_WS=0" | tr "\n" " ")"
  done
done
