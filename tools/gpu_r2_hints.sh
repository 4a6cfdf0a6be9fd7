mkdir -p gpurun_out
S=140,170,300
for H in 0 3 7; do
  for L in "c2 0" "c5 7"; do
    WF_WS_DISCARD=1 WF_WS_HINTS=$H timeout 300 python tools/ring_sweep.py $L $S
  done
done > gpurun_out/hints.jsonl 2>&1
cat gpurun_out/hints.jsonl
for H in 0 3 7; do
  WF_WS_DISCARD=1 WF_WS_HINTS=$H timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/hints_c2_h$H.csv \
    python tools/ring_sweep.py c2 0 $S --profile > /dev/null 2>&1
  WF_WS_DISCARD=1 WF_WS_HINTS=$H timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/hints_c5_h$H.csv \
    python tools/ring_sweep.py c5 7 $S --profile > /dev/null 2>&1
done
echo done
