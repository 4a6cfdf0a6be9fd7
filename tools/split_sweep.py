"""Sweep the persistent kernel's role split (WF_SPLIT: % of CTAs running only F items) and lags on c2."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from bench import layer_inputs
spec, t, x, w = layer_inputs("c2")
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
xd = torch.from_numpy(x).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ref = None
for cfg in sys.argv[1].split(";"):
    sp, lag, lag2 = cfg.split(",")
    os.environ["WF_SPLIT"] = sp; os.environ["WF_LAG"] = lag; os.environ["WF_LAG2"] = lag2
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
    ts = []
    for i in range(14):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); y = plan(xd); b.record(); b.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
    yh = y.cpu().numpy()
    if ref is None: ref = yh
    print(f"split={sp:>3}% lag={lag:>3} lag2={lag2:>3}: median {np.median(ts):7.1f} us  min {min(ts):7.1f}  "
          f"same={np.array_equal(yh, ref)}", flush=True)
    del plan
