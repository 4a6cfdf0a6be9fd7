mkdir -p gpurun_out
S=100,120,140,170,200,300
for D in 1 3; do
  WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c2 0 $S > gpurun_out/ring2_c2_d$D.jsonl 2>&1
  WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c2 0 $S --clean > gpurun_out/ring2c_c2_d$D.jsonl 2>&1
  WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c5 7 $S --clean > gpurun_out/ring2c_c5_d$D.jsonl 2>&1
done
cat gpurun_out/ring2*.jsonl
for D in 1 3; do
  WF_WS_DISCARD=$D timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ring2_c2_d$D.csv \
    python tools/ring_sweep.py c2 0 $S --profile > /dev/null 2>&1
  WF_WS_DISCARD=$D timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ring2_c5_d$D.csv \
    python tools/ring_sweep.py c5 7 $S --profile > /dev/null 2>&1
done
echo done
