for C in 2 4 8 16 32; do timeout 300 python bench.py --no-per-config --no-cpu-baseline --steps 20 --e2e-chunks $C 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d = json.loads(l); print('chunks', $C, 'e2e ms', round(d['e2e']['ms_per_step'], 3), 'TFLOP/s', round(d['e2e']['value'], 2))
"; done
timeout 120 python tools/pcie_probe.py
