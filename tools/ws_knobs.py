"""Time one fused layer through LayerPlan under several environment settings
(warp-specialised kernel knobs: WF_WS_BUDGET_MB, WF_WS_LAG, WF_WS_DISCARD,
WF_WS_DBG ...).

    python tools/ws_knobs.py B C Cp HW T  'K=V,K=V'  'K=V' ...     (T = 16: FFT-16)
"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
b, c, cp, hw, t = (int(v) for v in sys.argv[1:6])
dev = torch.device("cuda", 0)
spec = wf.LayerSpec(b, c, cp, hw, hw, 3, 1, 1)
w = (np.random.default_rng(0).standard_normal(spec.kernel_dims()) * np.sqrt(2 / (9 * c))).astype(np.float32)
fft = t == 16                       # T = 16: the FFT-16 transform
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis() if fft else wf.make_basis(t))
x = torch.rand(spec.input_dims(), device=dev) * 2 - 1
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for setting in sys.argv[6:] or [""]:
    kv = dict(e.split("=") for e in setting.split(",") if e)
    for k, v in kv.items():
        os.environ[k] = v
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, transform="fft" if fft else "winograd",
                                                    device=dev))
    ts = []
    for i in range(12):
        flush.zero_()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan(x); e.record(); e.synchronize()
        if i >= 2: ts.append(a.elapsed_time(e) * 1e3)
    print(f"{setting or 'default':40s} {np.median(ts):9.1f} us", flush=True)
    del plan
    for k in kv:
        os.environ.pop(k)
