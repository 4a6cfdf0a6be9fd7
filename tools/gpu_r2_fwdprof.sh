# full ncu capture of the pipelined forward kernel (c3 L9) and the position GEMM
timeout 200 python tools/layer_time.py c3 8 --engine three_stage --reps 3 > gpurun_out/lt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_pipe" -s 1 -c 1 -o gpurun_out/l9_fwd2 -f \
  python tools/layer_time.py c3 8 --engine three_stage --reps 3 > gpurun_out/ncu_full.log 2>&1; echo full $?
