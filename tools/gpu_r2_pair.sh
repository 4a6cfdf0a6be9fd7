# CTA-pair position GEMM: new tests (hang guard), full suite, timings
set -x
timeout 600 python -m pytest tests/test_gpu_pair.py -x -q 2>&1 | tail -5 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for L in "c3 4" "c3 5" "c3 7" "c3 8" "c3 10" "c3 11" "c4 1" "c4 2" "c4 3"; do
  WF_GEMM_PAIR=0 timeout 60 python tools/layer_time.py $L --reps 20
  timeout 60 python tools/layer_time.py $L --reps 20
done
