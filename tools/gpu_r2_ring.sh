# ring-budget sweep (timing; then DRAM bytes under ncu) for c2 and c5 64->64 @56 and c5 128@56
mkdir -p gpurun_out
S=32,48,64,80,100,140,200,300
for D in 1 3; do
  WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c2 0 $S > gpurun_out/ring_c2_d$D.jsonl 2>&1
  WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c5 7 $S > gpurun_out/ring_c5_64_56_d$D.jsonl 2>&1
  WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c5 10 $S > gpurun_out/ring_c5_128_56_d$D.jsonl 2>&1
done
cat gpurun_out/ring_*.jsonl
for D in 1 3; do
  WF_WS_DISCARD=$D timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ring_c2_d$D.csv \
    python tools/ring_sweep.py c2 0 $S --profile > /dev/null 2>&1
  WF_WS_DISCARD=$D timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ring_c5_d$D.csv \
    python tools/ring_sweep.py c5 7 $S --profile > /dev/null 2>&1
done
echo done
