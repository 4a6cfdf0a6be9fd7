mkdir -p gpurun_out
timeout 200 python tools/layer_time.py c4 0 --reps 2 > gpurun_out/lt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_|gemm_resident" -s 9 -c 3 -o gpurun_out/c4L1_full -f \
  python tools/layer_time.py c4 0 --reps 2 > gpurun_out/ncu_c4.log 2>&1; echo c4 $?
timeout 200 python tools/layer_time.py c3 8 --reps 2 > gpurun_out/lt2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_staged|position_gemm|inverse_vec" -s 9 -c 3 -o gpurun_out/c3L9_full -f \
  python tools/layer_time.py c3 8 --reps 2 > gpurun_out/ncu_c3.log 2>&1; echo c3 $?
