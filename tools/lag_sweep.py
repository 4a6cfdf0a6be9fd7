"""Sweep WF_LAG / WF_L2_BUDGET_MB of the static-order persistent kernel on c2."""
import os, sys, itertools
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
lags = [int(v) for v in sys.argv[1].split(",")]
budgets = [int(v) for v in sys.argv[2].split(",")]
for bud, lag in itertools.product(budgets, lags):
    os.environ["WF_LAG"] = str(lag); os.environ["WF_L2_BUDGET_MB"] = str(bud)
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
    ts = []
    for i in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan(xd); b.record(); b.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
    print(f"budget={bud:4d} lag={lag:3d}: median {np.median(ts):7.1f} us  min {min(ts):7.1f}", flush=True)
    del plan
