mkdir -p gpurun_out
for S3 in 0 1; do for rep in 1 2; do WF_WS_SLOTS3=$S3 timeout 300 python tools/ring_sweep.py c2 0 140; done; done 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d = json.loads(l); print(d['layer'][:24], d['median_us'], d['min_us'])
    else: print(l.rstrip()[:200])
"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "warp_specialised or c2 or instrumented or planned or mixed or concurrent" > gpurun_out/ws_tests.log 2>&1; tail -3 gpurun_out/ws_tests.log
