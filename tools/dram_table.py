"""DRAM bytes per layer, fused vs three-stage (SURVEY.md 8(d), row ⊕2).

Run under ncu (one pass, no cache flushing between the kernels of a call, so
L2 reuse across a call's kernels counts as it does in the bench):

    ncu --profile-from-start off --cache-control none --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/dram.csv python tools/dram_table.py [configs] > gpurun_out/dram_calls.jsonl
    python tools/dram_table.py --report gpurun_out/dram.csv gpurun_out/dram_calls.jsonl > profiles/rNN_dram_table.md

Profiling mode: for every layer of the configs and both engines, one warm
call, an L2 flush (a 256 MB write, then a 256 MB read so that no dirty
flush line is written back inside the measured call; outside the profiled
range), then ONE call inside
cudaProfilerStart/Stop; the call's kernel count (wf_kernel_launches) maps
the ncu rows back to layers.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def profile(configs):
    import torch
    import paper_1912_02165_b200 as wf
    from paper_1912_02165_b200 import _lib
    from bench import CONFIGS, roofline_terms
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for cfg in configs:
        for k, ld in enumerate(CONFIGS[cfg]):
            spec, x, w = ld.inputs()
            basis = wf.make_fft_basis(3) if ld.tile == 16 else wf.make_basis(ld.tile)
            pack = wf.transform_kernels(wf.Tensor4D(w), basis)
            xd = torch.from_numpy(x).to(dev)
            rt = roofline_terms(spec, ld.tile)
            for engine in ("fused", "three_stage"):
                plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind=engine, tile=ld.tile, transform=ld.transform,
                                                                device=dev))
                plan(xd)
                flush.zero_()
                flush.sum()          # read pass: the flush's dirty lines are written back now, not inside the call
                torch.cuda.synchronize()
                n0 = lib.wf_kernel_launches()
                torch.cuda.profiler.start()
                plan(xd)
                torch.cuda.synchronize()
                torch.cuda.profiler.stop()
                n = lib.wf_kernel_launches() - n0
                print(json.dumps({"config": cfg, "layer": ld.label(), "engine": engine, "launches": n,
                                  "variant": plan.variant or "three_stage", "q_fused": rt["q_fused"],
                                  "q_three": rt["q_three"]}), flush=True)
                del plan
            del xd
            torch.cuda.empty_cache()


def report(csv_path, calls_path):
    rows = {}
    with open(csv_path) as fh:
        text = fh.read()
    start = text.find('"ID"')
    for r in csv.DictReader(text[start:].splitlines()):
        kid = int(r["ID"])
        d = rows.setdefault(kid, {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)
        d[r["Metric Name"]] = v * scale
    kernels = [rows[k] for k in sorted(rows)]
    calls = [json.loads(ln) for ln in open(calls_path) if ln.startswith("{")]
    pos = 0
    print("| config | layer | engine (variant) | kernels | DRAM read MB | DRAM write MB | DRAM total MB | "
          "Q_fused MB | total / Q_fused | kernel time us |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    pairs = {}
    for c in calls:
        ks = kernels[pos:pos + c["launches"]]
        pos += c["launches"]
        rd = sum(k.get("dram__bytes_read.sum", 0) for k in ks)
        wr = sum(k.get("dram__bytes_write.sum", 0) for k in ks)
        t = sum(k.get("gpu__time_duration.sum", 0) for k in ks)
        pairs.setdefault((c["config"], c["layer"]), {})[c["engine"]] = (rd + wr, c)
        print(f"| {c['config']} | {c['layer']} | {c['engine']} ({c['variant']}) | {len(ks)} | {rd / 1e6:.1f} | "
              f"{wr / 1e6:.1f} | {(rd + wr) / 1e6:.1f} | {c['q_fused'] / 1e6:.1f} | {(rd + wr) / c['q_fused']:.2f} | "
              f"{t * 1e6:.1f} |")
    print()
    print("| config | layer | fused DRAM MB | three-stage DRAM MB | three-stage / fused | ideal Q_3stage / Q_fused |")
    print("|---|---|---|---|---|---|")
    traffic = {}
    for (cfg, layer), d in pairs.items():
        if "fused" in d and "three_stage" in d:
            f, c = d["fused"]
            s, _ = d["three_stage"]
            print(f"| {cfg} | {layer} | {f / 1e6:.1f} | {s / 1e6:.1f} | {s / max(f, 1):.2f} | "
                  f"{c['q_three'] / c['q_fused']:.2f} |")
            traffic.setdefault(cfg, {})[layer] = {"fused": int(f), "three_stage": int(s)}
    return traffic


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--report":
        t = report(sys.argv[2], sys.argv[3])
        if len(sys.argv) > 4:
            with open(sys.argv[4], "w") as fh:
                json.dump(t, fh, indent=1)
    else:
        profile(sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"])
