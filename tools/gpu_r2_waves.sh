# one-wave rule for pair-GEMM layers: tests + fused times
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for L in "c3 7" "c3 8" "c3 9" "c3 10" "c3 11" "c3 12" "c4 1"; do timeout 60 python tools/layer_time.py $L --reps 20; done
