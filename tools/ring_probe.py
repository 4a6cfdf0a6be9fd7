import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_1912_02165_b200 as wf
from test_gpu_parity import _fused_ex, _run, _he
for dims, t in [((24, 64, 64, 56, 56, 3, 1, 1), 6), ((96, 32, 32, 56, 56, 3, 1, 1), 8), ((128, 16, 16, 56, 56, 3, 1, 1), 8),
                ((8, 128, 128, 56, 56, 3, 1, 1), 8), ((8, 256, 256, 28, 28, 3, 1, 1), 6), ((8, 3, 64, 112, 112, 3, 1, 1), 6)]:
    spec = wf.LayerSpec(*dims); rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, spec.input_dims()).astype(np.float32)
    pack = wf.transform_kernels(wf.Tensor4D(_he(rng, spec)), wf.make_basis(t))
    ref, _ = _run("three_stage", x, pack, spec, t)
    for ring in (1 << 20, 4 << 20, 9 << 20):
        for lag in (0, 2, 1000):
            for gb in (0, 8):
                y, v = _fused_ex(x, pack, spec, t, variant="ws", ring_bytes=ring, lag=lag, gbatch=gb)
                ok = np.array_equal(y, ref)
                print(dims, t, "ring", ring >> 20, "lag", lag, "gb", gb, "->", v, "OK" if ok else "MISMATCH", flush=True)
                assert ok
print("ring probe ok")
