mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "3xfp16" > gpurun_out/fp16_tests.log 2>&1; tail -15 gpurun_out/fp16_tests.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
