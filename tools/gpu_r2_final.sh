# round-2 measurement pass: GPU tests, smoke, bench (ours + reference arm), DRAM table, launch list, c2 capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 300 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -c 300 gpurun_out/bench_ref.log
timeout 600 python bench.py --precision 3xfp16 --no-per-config --no-cpu-baseline > gpurun_out/bench_fp16.log 2>&1; tail -c 300 gpurun_out/bench_fp16.log
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
