mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; python tools/bench_summary.py gpurun_out/bench.log | head -12
timeout 300 python tools/ws_roles.py c2 0 > gpurun_out/roles.log 2>&1; cat gpurun_out/roles.log
timeout 600 python -m pytest tests/test_fft.py tests/test_gpu_configs.py -m gpu -q -x -k "c4 or fft" > gpurun_out/fft_tests.log 2>&1; tail -2 gpurun_out/fft_tests.log
