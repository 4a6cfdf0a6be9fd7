"""Small layers through every engine path and fused variant, for compute-sanitizer runs.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf  # noqa: E402
from oracle import oracle as O  # noqa: E402

# (dims, tile, transform, fused variants to force)
cases = [
    ((2, 64, 64, 20, 20, 3, 1, 1), 6, "winograd", ("ws", "itemq", "waves")),   # F(4x4,3x3), the c2 / VGG kernel
    ((1, 16, 16, 24, 24, 3, 1, 1), 8, "winograd", ("ws", "itemq", "waves")),   # F(6x6,3x3), the c5 kernel
    ((1, 3, 64, 20, 20, 3, 1, 1), 6, "winograd", ("ws",)),                     # RGB layer (K padding)
    ((2, 20, 24, 13, 11, 3, 1, 0), 6, "winograd", ("itemq", "waves")),          # ragged sizes, pad_hi 0
    ((1, 3, 16, 20, 20, 3, 1, 1), 4, "winograd", ("auto",)),                    # F(2x2,3x3)
    ((1, 64, 512, 12, 12, 3, 1, 1), 6, "winograd", ("waves",)),                # CTA-pair GEMM layer
    ((2, 3, 5, 16, 16, 3, 1, 1), 16, "fft", ("waves",)),
    ((1, 24, 40, 29, 31, 3, 0, 1), 16, "fft", ("waves",)),
]
for dims, t, tf, variants in cases:
    spec = wf.LayerSpec(*dims)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(spec.input_dims()).astype(np.float32)
    w = (rng.standard_normal(spec.kernel_dims()) * 0.1).astype(np.float32)
    basis = wf.make_fft_basis() if tf == "fft" else wf.make_basis(t)
    pack = wf.transform_kernels(wf.Tensor4D(w), basis)
    ref = O.direct_conv_f64(x, w, spec)
    runs = [("three_stage", "auto")] + [("fused", v) for v in variants]
    for kind, variant in runs:
        cfg = wf.EngineConfig(kind=kind, tile=t, transform=tf, fused_variant=variant)
        y, st = wf.run_engine(kind, wf.Tensor4D(x), pack, spec, cfg)
        err = O.max_rel_error(y.data, ref)
        assert err < 1e-3, (dims, t, tf, kind, variant, err)
        print(f"{dims} T={t} {tf} {kind}/{variant} -> ran {st.variant}: max_rel_err {err:.2e}", flush=True)
    wf.conv_direct(wf.Tensor4D(x), wf.Tensor4D(w), spec)
print("sanitize cases ok")
