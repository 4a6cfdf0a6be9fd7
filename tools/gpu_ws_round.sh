# measurement pass for the warp-specialised kernel: tests, bench (both arms),
# all configs, ncu launch list + one full capture of the c2 fused step
mkdir -p gpurun_out
make -s -j8 >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 1200 python tools/bench_all.py --reps 10 > gpurun_out/all_configs.md 2> gpurun_out/all_configs.err; echo all $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ws -s 3 -c 1 -o gpurun_out/ws_full -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2 $?
