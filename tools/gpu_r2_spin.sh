mkdir -p gpurun_out
for L in "c2 0" "c5 7" "c5 0" "c3 1" "c3 6"; do timeout 300 python tools/ring_sweep.py $L 140; done 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d = json.loads(l); print(d['layer'][:28], d['median_us'], d['min_us'])
    else: print(l.rstrip()[:200])
"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
