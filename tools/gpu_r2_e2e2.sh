mkdir -p gpurun_out
for c in 2 4 6 8 12 16; do
  timeout 300 python bench.py --no-per-config --no-cpu-baseline --steps 10 --warmup 3 --e2e-chunks $c > gpurun_out/e2e_$c.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/e2e_$c.log") if x.startswith("{")][-1]
d=json.loads(l); print("chunks", $c, "e2e ms", d["e2e"]["ms_per_step"], "value", d["e2e"]["value"])
PY
done
timeout 120 python tools/pcie_probe.py 2>&1 | tail -12
