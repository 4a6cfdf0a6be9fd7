"""Timeline of HostPipeline (per-slice H2D / compute / D2H end times) for c2."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
dev = torch.device("cuda", 0)
spec = wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1)
w = (np.random.default_rng(0).standard_normal(spec.kernel_dims()) * 0.06).astype(np.float32)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(6))
chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pipe = wf.HostPipeline(spec, pack, wf.EngineConfig(kind="fused", tile=6, device=dev), chunks=chunks, graph=False)
x = torch.randn(spec.input_dims()).pin_memory()
y = torch.empty(spec.output_dims()).pin_memory()
for _ in range(3): pipe(x, y)
torch.cuda.synchronize()
s_in, s_comp, s_out = pipe.streams
t0 = torch.cuda.Event(enable_timing=True)
cur = torch.cuda.current_stream()
t0.record(cur)
for s in pipe.streams: s.wait_stream(cur)
marks = []
for i, (lo, hi) in enumerate(pipe.bounds):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    with torch.cuda.stream(s_in):
        pipe.x_dev[lo:hi].copy_(x[lo:hi], non_blocking=True); pipe.ev_in[i].record(s_in); e[0].record(s_in)
    with torch.cuda.stream(s_comp):
        s_comp.wait_event(pipe.ev_in[i]); pipe.plans[hi - lo](pipe.x_dev[lo:hi], out=pipe.y_dev[lo:hi])
        pipe.ev_comp[i].record(s_comp); e[1].record(s_comp)
    with torch.cuda.stream(s_out):
        s_out.wait_event(pipe.ev_comp[i]); y[lo:hi].copy_(pipe.y_dev[lo:hi], non_blocking=True); e[2].record(s_out)
    marks.append(e)
torch.cuda.synchronize()
for i, e in enumerate(marks):
    print(i, " ".join(f"{t0.elapsed_time(ev) * 1e3:8.1f}" for ev in e), " (us: H2D done, compute done, D2H done)")
