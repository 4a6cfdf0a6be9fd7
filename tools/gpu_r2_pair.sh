# CTA-pair position GEMM: KS = 32 (6 stages) vs 64 (3 stages)
set -x
timeout 600 python -m pytest tests/test_gpu_pair.py -x -q 2>&1 | tail -2 || exit 1
WF_PAIR_KS=64 timeout 600 python -m pytest tests/test_gpu_pair.py -x -q 2>&1 | tail -2 || exit 1
for L in "c3 7" "c3 8" "c3 10"; do
  WF_PAIR_KS=64 timeout 60 python tools/layer_time.py $L --reps 20
  timeout 60 python tools/layer_time.py $L --reps 20
  WF_PAIR_KS=64 timeout 60 python tools/layer_time.py $L --engine three_stage --reps 20
  timeout 60 python tools/layer_time.py $L --engine three_stage --reps 20
done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/pair_launches.csv python tools/layer_time.py c3 8 --engine three_stage --reps 2
