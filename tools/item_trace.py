"""Timeline of the persistent kernel's items (WF_PROFILE=2): utilisation over time per kind."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["WF_PROFILE"] = "2"
import paper_1912_02165_b200 as wf
from paper_1912_02165_b200 import _lib
from bench import layer_inputs
spec, t, x, w = layer_inputs(sys.argv[1] if len(sys.argv) > 1 else "c2")
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
xd = torch.from_numpy(x).to(dev)
lib = _lib.load()
lib.wf_debug_fused_trace.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * (16384 * 2))()
for it in range(3):
    lib.wf_debug_fused_trace(buf, 16384)
    plan(xd); torch.cuda.synchronize()
    n = lib.wf_debug_fused_trace(buf, 16384)
a = np.array(buf[:2 * n], dtype=np.uint64).reshape(n, 2)
cta = (a[:, 0] >> 32).astype(np.int64)
kind = ((a[:, 0] >> 24) & 0xFF).astype(np.int64)
blk = (a[:, 0] & 0xFFFFFF).astype(np.int64)
start = (a[:, 1] & ((1 << 40) - 1)).astype(np.int64)
dur = (a[:, 1] >> 40).astype(np.int64)
t0 = start.min()
start -= t0
end = start + dur
T = end.max()
print(f"items {n}, span {T/1e3:.1f} us, CTAs {len(set(cta.tolist()))}")
bins = 20
edges = np.linspace(0, T, bins + 1)
ncta = len(set(cta.tolist()))
print("time(us)  busy%   F%   G%   I%   (share of CTA-time in each bin)   blocks F/G/I done by bin end")
for i in range(bins):
    lo, hi = edges[i], edges[i + 1]
    ov = np.clip(np.minimum(end, hi) - np.maximum(start, lo), 0, None)
    tot = ncta * (hi - lo)
    parts = [ov[kind == k].sum() / tot * 100 for k in range(3)]
    doneb = [len(set(blk[(kind == k) & (end <= hi)].tolist())) for k in range(3)]
    print(f"{hi/1e3:7.1f}  {sum(parts):5.1f}  {parts[0]:5.1f} {parts[1]:5.1f} {parts[2]:5.1f}   {doneb}")
for k, name in enumerate("FGI"):
    d = dur[kind == k]
    print(f"{name}: n={len(d)} mean {d.mean()/1e3:.2f} us  p50 {np.median(d)/1e3:.2f}  p90 {np.percentile(d,90)/1e3:.2f}")
