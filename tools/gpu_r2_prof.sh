# GPU tests + ncu evidence: DRAM bytes per layer (fused vs three-stage), c2 launch list, c2 full capture
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -8 gpurun_out/gpu_tests.log
timeout 280 python tools/dram_table.py > gpurun_out/dram_calls_plain.jsonl 2> gpurun_out/dram_plain.err && \
timeout 1200 ncu --profile-from-start off --cache-control none --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --csv --log-file gpurun_out/dram.csv python tools/dram_table.py > gpurun_out/dram_calls.jsonl 2> gpurun_out/dram_ncu.err; echo dram $?
timeout 300 python bench.py --no-per-config --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
  python bench.py --no-per-config --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches $?
timeout 200 python tools/layer_time.py c2 --reps 3 > gpurun_out/lt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ws -s 1 -c 1 -o gpurun_out/c2_ws_full -f \
  python tools/layer_time.py c2 --reps 3 > gpurun_out/ncu_full.log 2>&1; echo full $?
