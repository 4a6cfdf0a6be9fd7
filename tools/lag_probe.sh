# bounded probe of extreme lags on the batched-publish (narrow) layers: every run under a hard timeout
for l in "c5 1" "c5 2" "c5 3" "c5 4" "c5 5"; do
  for lag in 64 96 200; do
    echo -n "$l lag $lag: "
    out=$(WF_WS_LAG=$lag timeout -s KILL 25 python tools/layer_time.py $l --reps 3 2>&1 | tail -1)
    echo "${out:-KILLED (hang)}" | sed 's/.*median \([0-9.]*\) us.*/\1 us/'
  done
done
