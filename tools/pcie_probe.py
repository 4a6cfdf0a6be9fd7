"""Pinned host <-> device copy bandwidth: H2D alone, D2H alone, both concurrently (c2-sized buffers)."""
import torch, time
dev = torch.device("cuda", 0)
n = 51380224 // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, device=dev); d_b = torch.empty(n, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    d_a.copy_(h_in, non_blocking=True)
def d2h():
    h_out.copy_(d_b, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn in [("H2D", h2d), ("D2H", d2h), ("both", both)]:
    ms = timed(fn)
    gb = (2 if name == "both" else 1) * n * 4 / 1e9
    print(f"{name}: {ms:.3f} ms  {gb / ms * 1e3:.1f} GB/s aggregate")
