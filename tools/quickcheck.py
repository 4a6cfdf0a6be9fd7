"""Quick GPU parity check of the three engines vs an FP64 numpy direct conv."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
import torch

def direct64(x, w, spec):
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (spec.pad_lo, spec.pad_hi), (spec.pad_lo, spec.pad_hi)))
    out = np.zeros(spec.output_dims())
    for ky in range(3):
        for kx in range(3):
            out += np.einsum("bcyx,oc->boyx", xp[:, :, ky:ky + spec.out_height, kx:kx + spec.out_width], w[:, :, ky, kx].astype(np.float64))
    return out

def rel(a, b):
    return float(np.abs(a.astype(np.float64) - b).max() / max(np.abs(b).max(), 1e-30))

rng = np.random.default_rng(0)
cases = [(wf.LayerSpec(1, 8, 8, 9, 9, 3, 1, 1), 4), (wf.LayerSpec(2, 20, 24, 13, 11, 3, 1, 0), 6),
         (wf.LayerSpec(1, 64, 64, 56, 56, 3, 1, 1), 4), (wf.LayerSpec(2, 64, 64, 56, 56, 3, 1, 1), 6),
         (wf.LayerSpec(1, 3, 64, 32, 32, 3, 1, 1), 6), (wf.LayerSpec(1, 16, 16, 28, 28, 3, 1, 1), 8),
         (wf.LayerSpec(1, 130, 300, 14, 14, 3, 1, 1), 6), (wf.LayerSpec(1, 32, 32, 20, 20, 3, 0, 1), 5),
         (wf.LayerSpec(1, 32, 32, 20, 20, 3, 1, 1), 7)]
ok = True
for spec, T in cases:
    x = rng.standard_normal(spec.input_dims()).astype(np.float32)
    w = (rng.standard_normal(spec.kernel_dims()) * np.sqrt(2.0 / (9 * spec.in_channels))).astype(np.float32)
    ref = direct64(x, w, spec)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(T))
    d, _ = wf.conv_direct(wf.Tensor4D(x), wf.Tensor4D(w), spec)
    s, ss = wf.conv_three_stage(wf.Tensor4D(x), pack, spec, wf.EngineConfig(kind="three_stage", tile=T))
    f, fs = wf.conv_fused(wf.Tensor4D(x), pack, spec, wf.EngineConfig(kind="fused", tile=T))
    e = (rel(d.data, ref), rel(s.data, ref), rel(f.data, ref))
    same = np.array_equal(s.data, f.data)
    good = e[0] < 1e-6 and e[1] < 1e-3 and e[2] < 1e-3 and same
    ok &= good
    print(f"{spec} T={T}: direct {e[0]:.2e} three {e[1]:.2e} fused {e[2]:.2e} fused==three {same} "
          f"t3={ss.wall_s*1e6:.0f}us tf={fs.wall_s*1e6:.0f}us {'OK' if good else 'FAIL'}", flush=True)
print("QUICKCHECK", "PASS" if ok else "FAIL")
