mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "fft or c4 or 3xfp16" > gpurun_out/fft_tests.log 2>&1; tail -3 gpurun_out/fft_tests.log
for L in 0 1 2 3; do timeout 300 python tools/layer_time.py c4 $L; done
timeout 200 python tools/layer_time.py c2 --reps 3 > gpurun_out/lt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ws -s 1 -c 1 -o gpurun_out/c2_ws_full2 -f \
  python tools/layer_time.py c2 --reps 3 > gpurun_out/ncu_full.log 2>&1; echo full $?
