# FFT kernels: parity + c4 layer times + launch list of L1
set -x
timeout 600 python -m pytest tests/test_fft.py tests/test_gpu_pair.py -x -q 2>&1 | tail -2 || exit 1
for L in 0 1 2 3; do timeout 60 python tools/layer_time.py c4 $L --engine three_stage --reps 10; timeout 60 python tools/layer_time.py c4 $L --reps 10; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/fft_launches.csv python tools/layer_time.py c4 0 --engine three_stage --reps 2 > /dev/null 2>&1
