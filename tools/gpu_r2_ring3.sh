mkdir -p gpurun_out
S=140,170,300
for D in 1 3; do
  for L in "c2 0" "c5 7" "c5 10" "c5 2" "c3 0" "c3 1" "c3 3"; do
    WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py $L $S
  done
done > gpurun_out/ring3.jsonl 2>&1
cat gpurun_out/ring3.jsonl
for D in 1 3; do
  WF_WS_DISCARD=$D timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ring3_c2_d$D.csv \
    python tools/ring_sweep.py c2 0 $S --profile > /dev/null 2>&1
done
echo done
