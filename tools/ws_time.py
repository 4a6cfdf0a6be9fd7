"""c2 (or a given config): warp-specialised kernel (WF_WS=1) vs the item-queue
persistent kernel (WF_WS=0): bitwise comparison and CUDA-event timing (L2 flushed).

    python tools/ws_time.py [config] [reps] [env=val ...]
"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from bench import layer_inputs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    os.environ[k] = v
spec, t, x, w = layer_inputs(cfg)
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
xd = torch.from_numpy(x).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
outs = {}
for ws in ("0", "1"):
    os.environ["WF_WS"] = ws
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); y = plan(xd); b.record(); b.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
    outs[ws] = y.clone()
    print(f"WF_WS={ws}: median {np.median(ts):7.1f} us  min {np.min(ts):7.1f}", flush=True)
d = (outs["0"] - outs["1"]).abs().max().item()
print("bitwise equal" if torch.equal(outs["0"], outs["1"]) else f"DIFFER max abs {d:.3e}")
