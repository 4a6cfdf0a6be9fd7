"""FFT-16 overlap-save variant (BASELINE config c4).

The reference has no FFT path, so there are no reference
golden vectors: FFT parity is anchored on the FP64 direct oracle only
("parity unpinned" against the reference).  CPU tests check the
pack expansion and the overlap-save tiling through the numpy FP64
restatement ``oracle.fft_conv_f64``; GPU tests check the sm_100a kernels.

Tolerance: max|y - y_fp64| / max|y_fp64| <= 1e-3 (3xbf16); the single-pass
bf16 mode has a looser documented bound (TOL_FFT_BF16).
"""
import numpy as np
import pytest

import paper_1912_02165_b200 as wf
from oracle import oracle as O

TOL_FFT = 1e-3
TOL_FFT_BF16 = 2e-2


def _case(dims, seed=0):
    spec = wf.LayerSpec(*dims)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(spec.input_dims()).astype(np.float32)
    w = (rng.standard_normal(spec.kernel_dims()) * np.sqrt(2.0 / (9 * spec.in_channels))).astype(np.float32)
    return spec, x, w


# ------------------------------------------------------------------- CPU
@pytest.mark.parametrize("dims", [
    (1, 1, 1, 5, 5, 3, 1, 1),
    (2, 3, 5, 16, 16, 3, 1, 1),
    (1, 4, 2, 29, 31, 3, 0, 1),
    (1, 2, 3, 14, 14, 3, 1, 1),
])
def test_fft_restatement_matches_direct_fp64(dims):
    spec, x, w = _case(dims)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis(3))
    assert pack.transform == "fft" and pack.data.shape == (144, 2 * spec.in_channels, 2 * spec.out_channels)
    got = O.fft_conv_f64(x, pack.data, spec)
    ref = O.direct_conv_f64(x, w, spec)
    assert got.shape == ref.shape
    assert O.max_rel_error(got, ref) <= 1e-6   # pack is f32-rounded; the rest is f64


def test_fft_pack_block_structure():
    _, _, w = _case((1, 3, 4, 8, 8, 3, 1, 1), seed=3)
    d = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis()).data
    c, cp = 3, 4
    assert np.array_equal(d[:, :c, :cp], d[:, c:, cp:])          # Re V on both diagonal blocks
    assert np.array_equal(d[:, :c, cp:], -d[:, c:, :cp])         # Im V / -Im V
    assert np.all(d[0, :c, cp:] == 0) and np.all(d[0, c:, :cp] == 0)   # DC bin is real


def test_fft_config_and_pack_validation():
    spec, x, w = _case((1, 2, 2, 9, 9, 3, 1, 1))
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(transform="fft", tile=8)
    wpack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(6))
    cfg = wf.EngineConfig(kind="fused", transform="fft", tile=16)
    with pytest.raises(wf.ShapeMismatchError):                    # a Winograd pack under an FFT config
        wf.conv_fused(wf.Tensor4D(x), wpack, spec, cfg)
    assert wf.multiply_flops(10, 2, 3, 16, "fft") == 8 * 10 * 2 * 3 * 144


# ------------------------------------------------------------------- GPU
C4_REDUCED = [  # BASELINE c4 shapes (C = C', H = W), batch reduced from 128 for the FP64 oracle
    (64, 56, 4), (128, 28, 4), (256, 14, 2), (512, 7, 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("c,hw,b", C4_REDUCED)
def test_fft_config4_shapes_vs_fp64(c, hw, b):
    spec, x, w = _case((b, c, c, hw, hw, 3, 1, 1), seed=c)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis())
    ref = O.direct_conv_f64(x, w, spec)
    for kind in ("fused", "three_stage"):
        cfg = wf.EngineConfig(kind=kind, transform="fft", tile=16)
        out, stats = wf.run_engine(kind, wf.Tensor4D(x), pack, spec, cfg)
        err = O.max_rel_error(out.data, ref)
        assert err <= TOL_FFT, (kind, c, hw, err)
        assert stats.transform == "fft" and stats.flops == 8 * stats.n_tile * c * c * 144


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [
    (1, 1, 1, 1, 1, 3, 1, 1),        # single pixel, pure padding
    (2, 3, 5, 16, 16, 3, 1, 1),      # C, C' not multiples of 8 (element-wise slab path + K padding)
    (1, 4, 2, 29, 31, 3, 0, 1),      # asymmetric padding, ragged tiles
    (3, 8, 24, 30, 15, 3, 1, 1),     # several partial tile rows/columns
    (1, 130, 20, 20, 20, 3, 1, 1),   # several K blocks with padding
])
def test_fft_edge_shapes(dims):
    spec, x, w = _case(dims, seed=7)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis())
    ref = O.direct_conv_f64(x, w, spec)
    f, _ = wf.conv_fused(wf.Tensor4D(x), pack, spec, wf.EngineConfig(transform="fft", tile=16))
    s, _ = wf.conv_three_stage(wf.Tensor4D(x), pack, spec,
                               wf.EngineConfig(kind="three_stage", transform="fft", tile=16))
    assert np.array_equal(f.data, s.data)           # same kernels, same order: bitwise
    assert O.max_rel_error(f.data, ref) <= TOL_FFT
    assert O.max_rel_error(f.data, O.fft_conv_f64(x, pack.data, spec)) <= TOL_FFT


@pytest.mark.gpu
def test_fft_bf16_single_pass_bound():
    spec, x, w = _case((2, 64, 64, 28, 28, 3, 1, 1), seed=11)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis())
    out, _ = wf.conv_fused(wf.Tensor4D(x), pack, spec,
                           wf.EngineConfig(transform="fft", tile=16, precision="bf16"))
    assert O.max_rel_error(out.data, O.direct_conv_f64(x, w, spec)) <= TOL_FFT_BF16


@pytest.mark.gpu
def test_fft_torch_cuda_weights_and_layer_plan(cuda_dev):
    import torch
    spec, x, w = _case((2, 16, 32, 30, 30, 3, 1, 1), seed=5)
    pack = wf.transform_kernels(torch.from_numpy(w).to(cuda_dev), wf.make_fft_basis())
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(transform="fft", tile=16, device=cuda_dev))
    y = plan(torch.from_numpy(x).to(cuda_dev))
    torch.cuda.synchronize()
    assert O.max_rel_error(y.cpu().numpy(), O.direct_conv_f64(x, w, spec)) <= TOL_FFT
