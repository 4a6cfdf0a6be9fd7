"""Small layers through every engine path, for compute-sanitizer runs."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from oracle import oracle as O
cases = [((2, 20, 24, 13, 11, 3, 1, 0), 6, "winograd"), ((1, 3, 16, 20, 20, 3, 1, 1), 4, "winograd"),
         ((2, 64, 64, 30, 28, 3, 1, 1), 6, "winograd"), ((1, 16, 16, 20, 20, 3, 1, 1), 8, "winograd"),
         ((2, 3, 5, 16, 16, 3, 1, 1), 16, "fft"), ((1, 24, 40, 29, 31, 3, 0, 1), 16, "fft")]
for force in ("0", "1"):
    os.environ["WF_PERSIST_MIN_BLOCKS"] = "1" if force == "1" else "16"
    for dims, t, tf in cases:
        spec = wf.LayerSpec(*dims)
        rng = np.random.default_rng(0)
        x = rng.standard_normal(spec.input_dims()).astype(np.float32)
        w = (rng.standard_normal(spec.kernel_dims()) * 0.1).astype(np.float32)
        basis = wf.make_fft_basis() if tf == "fft" else wf.make_basis(t)
        pack = wf.transform_kernels(wf.Tensor4D(w), basis)
        ref = O.direct_conv_f64(x, w, spec)
        for kind in ("fused", "three_stage"):
            y, _ = wf.run_engine(kind, wf.Tensor4D(x), pack, spec, wf.EngineConfig(kind=kind, tile=t, transform=tf))
            err = O.max_rel_error(y.data, ref)
            assert err < 1e-3, (dims, t, tf, kind, err)
        d, _ = wf.conv_direct(wf.Tensor4D(x), wf.Tensor4D(w), spec)
print("sanitize cases ok")
