mkdir -p gpurun_out
timeout 200 python tools/layer_time.py c5 7 --reps 3 > gpurun_out/lt5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ws -s 1 -c 1 -o gpurun_out/c5_ws -f \
  python tools/layer_time.py c5 7 --reps 3 > gpurun_out/ncu_full5.log 2>&1; echo full $?
