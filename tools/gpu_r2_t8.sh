mkdir -p gpurun_out
for D in 0 1 2 3; do
  WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c5 7 140
  WF_WS_DISCARD=$D WF_LIB_PATH=build/ab/libT8h.so timeout 300 python tools/ring_sweep.py c5 7 140
done > gpurun_out/t8.jsonl 2>&1; cat gpurun_out/t8.jsonl
for D in 0 1 2 3; do
  for L in "" "build/ab/libT8h.so"; do
    WF_WS_DISCARD=$D WF_LIB_PATH=$L timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/t8_d${D}_$(basename ${L:-base}).csv \
      python tools/ring_sweep.py c5 7 140 --profile > /dev/null 2>&1
  done
done
# c2 with hints (T6 default) for the record, discard 1 vs 0
for D in 0 1; do WF_WS_DISCARD=$D timeout 300 python tools/ring_sweep.py c2 0 140,170; done
echo done
