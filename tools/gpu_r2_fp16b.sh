mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for L in 4 8 16 32 64; do WF_WS_LAG=$L timeout 300 python tools/ring_sweep.py c5 0 140; WF_WS_LAG=$L timeout 300 python tools/ring_sweep.py c5 3 140; WF_WS_LAG=$L timeout 300 python tools/ring_sweep.py c5 9 140; done 2>&1 | python3 -c "
import sys, json, os
for l in sys.stdin:
    if l.startswith('{'): d = json.loads(l); print(d['layer'][:24], d['median_us'])
    else: print(l.rstrip()[:150])
"
