"""Sweep the persistent kernel's scheduling knobs (env WF_P0, WF_NU) on c2."""
import os, sys, itertools
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from bench import layer_inputs
spec, t, x, w = layer_inputs("c2")
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
xd = torch.from_numpy(x).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
p0s = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "6,9,11,14,18").split(",")]
nus = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "21,28").split(",")]
for nu, p0 in itertools.product(nus, p0s):
    os.environ["WF_P0"] = str(p0); os.environ["WF_NU"] = str(nu)
    ts = []
    for i in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan(xd); b.record(); b.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
    print(f"NU={nu:3d} P0={p0:3d}: median {np.median(ts):7.1f} us  min {min(ts):7.1f}", flush=True)
