"""Summarise a bench.py JSON line (headline + per-config per-layer table) as markdown.

    python tools/bench_summary.py gpurun_out/bench.log > profiles/rNN_bench_summary.md
"""
import json
import sys

line = [l for l in open(sys.argv[1]) if l.startswith("{")][-1]
d = json.loads(line)
r = d["roofline"]
print(f"# bench.py headline ({d['config']['workload']})\n")
print(f"- value **{d['value']:.1f} {d['unit']}**, {d['ms_per_step'] * 1e3:.1f} us/step (mean of {d['steps']}), "
      f"roofline {r['bound']} {r['achieved']:.0f} / {r['peak']:.0f} {r['unit']} = **{r['frac']:.3f}**, "
      f"traffic {r['traffic']}")
e = d["e2e"]
print(f"- e2e {e['value']:.2f} {e['unit']} ({e['ms_per_step']:.3f} ms/step, {e['api']})")
c = d.get("cpu_baseline") or {}
c3 = d.get("cpu_baseline_three_stage") or {}
print(f"- CPU baseline (reference algorithm, {c.get('cores')} threads): fused {c.get('value') or 0:.3f} TFLOP/s, "
      f"three-stage {c3.get('value') or 0:.3f} TFLOP/s ({c.get('sample', '')[:160]})")
print(f"- clocks {d['clocks']}, gpu_launches {d['gpu_launches']}\n")
rows = [("headline", d["config"]["workload"], d["ms_per_step"], d["value"], d.get("layers", []))]
for k, v in d.get("per_config", {}).items():
    rows.append((k, v["workload"], v["ms_per_step"], v["value"], v["layers"]))
print("| config | layer | B | variant | fused ms | three-stage ms | fused speedup | TFLOP/s | t_roof us | bound | roofline frac |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for name, wl, ms, val, layers in rows:
    for L in layers:
        print(f"| {name} | {L['layer']} | {L['B']} | {L.get('variant')} | {L['ms']:.4f} | {L.get('three_stage_ms', '-')} | "
              f"{L.get('fused_speedup', '-')} | {L['tflops']} | {L['t_roof_us']} | {L['bound']} | {L['roofline_frac']} |")
print()
print("| config | ms per step (all layers) | TFLOP/s | three-stage ms |")
print("|---|---|---|---|")
for k, v in d.get("per_config", {}).items():
    print(f"| {k} | {v['ms_per_step']:.3f} | {v['value']:.1f} | {v['three_stage_ms_per_step']:.3f} |")
