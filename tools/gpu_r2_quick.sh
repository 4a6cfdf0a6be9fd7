# quick check after a ws-kernel change: a few layer times, then the GPU parity tests
mkdir -p gpurun_out
for a in "c2 0" "c3 1" "c3 3" "c3 5" "c5 4" "c5 7" "c5 10"; do timeout 200 python tools/layer_time.py $a --reps 20 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
