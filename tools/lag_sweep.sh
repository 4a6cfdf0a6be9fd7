# bounded lag sweep (WF_WS_LAG; 0 = the default rule), every run under a hard timeout
for l in "c2 0" "c3 1" "c3 3" "c3 4" "c3 5" "c5 3" "c5 4" "c5 5" "c5 6" "c5 7" "c5 8" "c5 9" "c5 10" "c5 11"; do
  echo -n "$l:"
  for lag in 0 6 8 12 16 24 32 48; do
    t=$(WF_WS_LAG=$lag timeout -s KILL 40 python tools/layer_time.py $l --reps 6 2>&1 | tail -1 | sed 's/.*median \([0-9.]*\) us.*/\1/')
    echo -n " $lag=${t:-KILLED}"
  done
  echo
done
