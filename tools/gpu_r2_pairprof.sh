timeout 200 python tools/layer_time.py c3 8 --engine three_stage --reps 3 > gpurun_out/lt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"position_gemm" -s 1 -c 1 -o gpurun_out/l9_pair -f \
  python tools/layer_time.py c3 8 --engine three_stage --reps 3 > gpurun_out/ncu_full.log 2>&1; echo full $?
