timeout 200 python tools/layer_time.py c2 --reps 3 > gpurun_out/lt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ws -s 1 -c 1 -o gpurun_out/c2_ws -f \
  python tools/layer_time.py c2 --reps 3 > gpurun_out/ncu_full.log 2>&1; echo full $?
