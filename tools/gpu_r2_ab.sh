mkdir -p gpurun_out
for rep in 1 2; do
  WF_LIB_PATH=build/ab/libB.so timeout 300 python tools/ring_sweep.py c2 0 140,300
  timeout 300 python tools/ring_sweep.py c2 0 140,300
  WF_LIB_PATH=build/ab/libB.so timeout 300 python tools/ring_sweep.py c5 7 140,300
  timeout 300 python tools/ring_sweep.py c5 7 140,300
done
timeout 300 python tools/ring_sweep.py c3 1 140,300
WF_LIB_PATH=build/ab/libB.so timeout 300 python tools/ring_sweep.py c3 1 140,300
timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ab_c2.csv \
    python tools/ring_sweep.py c2 0 140,300 --profile > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ab_c5.csv \
    python tools/ring_sweep.py c5 7 140,300 --profile > /dev/null 2>&1
echo done
