# F/I worker halves in the warp-specialised kernel: parity, then time vs the build without
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_specialised or golden or config2 or config3 or config5 or instrumented" 2>&1 | tail -2 || exit 1
for L in "c2 0" "c3 1" "c3 3" "c3 0" "c5 4"; do
  WF_LIB_PATH=build_alt/libwinofuse_b200.so timeout 60 python tools/layer_time.py $L --reps 20
  timeout 60 python tools/layer_time.py $L --reps 20
done
timeout 120 python tools/ws_roles.py c2 0 2>&1 | tail -26
