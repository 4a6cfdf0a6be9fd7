# c2: per-role accounting + ncu full capture with source
mkdir -p gpurun_out
timeout 200 python tools/ws_roles.py c2 0 > gpurun_out/roles_c2.log 2>&1; tail -40 gpurun_out/roles_c2.log
timeout 200 python tools/layer_time.py c2 --reps 3 > gpurun_out/lt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ws -s 1 -c 1 -o gpurun_out/c2_ws -f \
  python tools/layer_time.py c2 --reps 3 > gpurun_out/ncu_full.log 2>&1; echo full $?
