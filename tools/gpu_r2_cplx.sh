mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fft.py tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -q -x -k "fft or c4 or golden" > gpurun_out/cplx_tests.log 2>&1; tail -3 gpurun_out/cplx_tests.log
for L in 0 1 2 3; do timeout 300 python tools/layer_time.py c4 $L; timeout 300 python tools/layer_time.py c4 $L --engine three_stage; done
