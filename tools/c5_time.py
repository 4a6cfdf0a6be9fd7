"""Time the c5 sweep's F(6x6,3x3) layers (B = 256) through LayerPlan, with the
warp-specialised kernel and with the item-queue kernel (WF_WS=0).

    python tools/c5_time.py [C,...] [H,...]
"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
dev = torch.device("cuda", 0)
cs = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "64,128").split(",")]
hs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "28,56,112").split(",")]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for c in cs:
    for h in hs:
        spec = wf.LayerSpec(256, c, c, h, h, 3, 1, 1)
        w = (np.random.default_rng(0).standard_normal(spec.kernel_dims()) * np.sqrt(2 / (9 * c))).astype(np.float32)
        pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(8))
        x = torch.rand(spec.input_dims(), device=dev) * 2 - 1
        res = {}
        for ws in ("1", "0"):
            os.environ["WF_WS"] = ws
            plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=8, device=dev))
            ts = []
            for i in range(12):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); y = plan(x); b.record(); b.synchronize()
                if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
            res[ws] = (np.median(ts), y.clone())
            del plan
        same = torch.equal(res["1"][1], res["0"][1])
        print(f"c5 {c}->{c} @{h}: ws {res['1'][0]:8.1f} us   item-queue {res['0'][0]:8.1f} us   bitwise {same}", flush=True)
os.environ.pop("WF_WS")
