mkdir -p gpurun_out
for L in "c2 0" "c5 7" "c5 0" "c5 11" "c3 0" "c3 1" "c3 3" "c3 6"; do timeout 300 python tools/ring_sweep.py $L 140; done > gpurun_out/defaults.jsonl 2>&1
cat gpurun_out/defaults.jsonl
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 280 python tools/dram_table.py > gpurun_out/dram_calls_plain.jsonl 2> gpurun_out/dram_plain.err && \
timeout 1200 ncu --profile-from-start off --cache-control none --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --csv --log-file gpurun_out/dram.csv python tools/dram_table.py > gpurun_out/dram_calls.jsonl 2> gpurun_out/dram_ncu.err; echo dram $?
