# ncu --set full captures of the wave-path stage kernels (VGG 512->512 @28, FFT-16 64->64 @56)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:position_gemm_pair -s 2 -c 1 -o gpurun_out/l9_gemm -f python tools/layer_time.py c3 8 --reps 2 > gpurun_out/n1.log 2>&1; echo gemm $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:forward_pipe -s 2 -c 1 -o gpurun_out/l9_fwd -f python tools/layer_time.py c3 8 --reps 2 > gpurun_out/n2.log 2>&1; echo fwd $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:inverse_vec -s 2 -c 1 -o gpurun_out/l9_inv -f python tools/layer_time.py c3 8 --reps 2 > gpurun_out/n3.log 2>&1; echo inv $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_forward -s 3 -c 1 -o gpurun_out/c4_fftf -f python tools/layer_time.py c4 0 --reps 2 > gpurun_out/n4.log 2>&1; echo fftf $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_inverse -s 3 -c 1 -o gpurun_out/c4_ffti -f python tools/layer_time.py c4 0 --reps 2 > gpurun_out/n5.log 2>&1; echo ffti $?
