"""Ring-budget sweep of the warp-specialised fused kernel: time per ring size
(CUDA events, L2 flushed) and, under ncu, the DRAM bytes of one call each.

    python tools/ring_sweep.py c2 0 40,60,80,120,300          # timing
    ncu --profile-from-start off --cache-control none --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file out.csv \
        python tools/ring_sweep.py c2 0 40,60,80,120,300 --profile
WF_WS_DISCARD (env, read once per process) selects which consumed ring
lines are dropped from L2 (bit 1: U, bit 2: M).
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02165_b200 as wf  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg_name, layer, sizes = sys.argv[1], int(sys.argv[2]), [int(v) for v in sys.argv[3].split(",")]
profile = "--profile" in sys.argv
clean = "--clean" in sys.argv          # timing with a write + read flush (no dirty flush lines in L2)
ld = CONFIGS[cfg_name][layer]
spec, x, w = ld.inputs()
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(ld.tile))
xd = torch.from_numpy(x).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ref = None
for mb in sizes:
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=ld.tile, device=dev, fused_variant="ws",
                                                    ring_bytes=mb << 20))
    y = plan(xd).clone()
    ref = y if ref is None else ref
    same = bool(torch.equal(y, ref))
    if profile:
        flush.zero_()
        flush.sum()              # clean L2: the flush's dirty lines are written back before the call
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        plan(xd)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"ring_mb": mb}), flush=True)
        continue
    ts = []
    for i in range(23):
        flush.zero_()
        if clean:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan(xd)
        e1.record()
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(json.dumps({"layer": ld.label(), "ring_mb": mb, "scratch_mb": round(plan.nbytes / 2**20, 1),
                      "median_us": round(statistics.median(ts), 1), "min_us": round(min(ts), 1),
                      "bitwise_equal_to_first": same, "discard": os.environ.get("WF_WS_DISCARD", "default"), "clean_flush": clean}),
          flush=True)
    del plan
