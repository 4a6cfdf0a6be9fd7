"""Parity at the stated sizes of every benchmarked config (BASELINE.json
configs c2-c5), through the exact path bench.py times (LayerPlan /
LayerStack with the default variant, rings, lags and publish batches).

* c2: all 64 images against the CPU oracle's FP64 direct convolution, and
  4 images against the reference's own f32 fused algorithm (the bit-exact C
  port, oracle/winofuse_oracle.c).
* c3 (13 VGG layers, B=32), c4 (FFT-16, B=128), c5 (F(6x6,3x3), B=256): per
  layer the full batch bitwise against the three-stage engine (on the
  device) and a seeded random subset of 4 images against FP64 direct
  (reference convention bench.py:154-168: a subset verifies a batch).
* c3 chained: every LayerStack segment (layers whose shapes chain) against
  the layer-by-layer FP64 oracle chain on 2 images.

Tolerance (north star): max|y - y_fp64| / max|y_fp64| <= 1e-3 per layer, 3xbf16.
"""
import numpy as np
import pytest

import paper_1912_02165_b200 as wf
from bench import CONFIGS
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _dev():
    import torch
    return torch.device("cuda", 0)


def _plan(ld, spec, w, kind):
    basis = wf.make_fft_basis(3) if ld.tile == 16 else wf.make_basis(ld.tile)
    pack = wf.transform_kernels(wf.Tensor4D(w), basis)
    cfg = wf.EngineConfig(kind=kind, tile=ld.tile, transform=ld.transform, device=_dev())
    return pack, wf.LayerPlan(spec, pack, cfg)


def _subset(batch, seed, k=4):
    return sorted(np.random.default_rng(seed).choice(batch, size=min(k, batch), replace=False).tolist())


def _check_layer(ld):
    import torch
    spec, x, w = ld.inputs()
    pack, fused = _plan(ld, spec, w, "fused")
    _, three = _plan(ld, spec, w, "three_stage")
    xd = torch.from_numpy(x).to(_dev())
    yf = fused(xd).clone()
    ys = three(xd)
    assert torch.equal(yf, ys), (ld.label(), "fused != three-stage")
    idx = _subset(spec.batch, ld.seed)
    sub = wf.LayerSpec(len(idx), spec.in_channels, spec.out_channels, spec.height, spec.width, 3, 1, 1)
    ref = O.direct_conv_f64(x[idx], w, sub)
    err = O.max_rel_error(yf[idx].cpu().numpy(), ref)
    assert err <= TOL, (ld.label(), idx, err)
    return fused.variant, err


def test_c2_full_batch_against_fp64_and_reference_f32():
    import torch
    ld = CONFIGS["c2"][0]
    spec, x, w = ld.inputs()
    pack, plan = _plan(ld, spec, w, "fused")
    assert plan.variant == "ws"
    y = plan(torch.from_numpy(x).to(_dev())).cpu().numpy()
    err = O.max_rel_error(y, O.direct_conv_f64(x, w, spec))          # all 64 images
    assert err <= TOL, err
    sub = wf.LayerSpec(4, 64, 64, 56, 56, 3, 1, 1)
    ref32 = O.conv_fused(x[:4], pack.data, sub, 6, 24, threads=O.threads())
    assert O.max_rel_error(y[:4], ref32) <= TOL


@pytest.mark.parametrize("k", range(13))
def test_c3_vgg_layer_at_b32(k):
    _check_layer(CONFIGS["c3"][k])


def test_c3_vgg_chained_segments_against_oracle_chain():
    """LayerStack segments of the VGG stack (shapes that chain without
    pooling) on the full B=32 batch; images 0 and 17 of the chain's output
    against the FP64 oracle applied layer by layer (f32 between layers)."""
    import torch
    layers = CONFIGS["c3"]
    segs, cur = [], [0]
    for i in range(1, len(layers)):
        if layers[i - 1].cp == layers[i].c and layers[i - 1].hw == layers[i].hw:
            cur.append(i)
        else:
            segs.append(cur)
            cur = [i]
    segs.append(cur)
    assert [len(s) for s in segs] == [2, 2, 3, 3, 3]
    for seg in segs:
        specs, packs, ws = [], [], []
        for i in seg:
            spec, x_i, w = layers[i].inputs()
            specs.append(spec)
            ws.append(w)
            packs.append(wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(6)))
            if i == seg[0]:
                x = x_i
        stack = wf.LayerStack(specs, packs, [wf.EngineConfig(kind="fused", tile=6, device=_dev())] * len(seg))
        y = stack(torch.from_numpy(x).to(_dev()))
        idx = [0, 17]
        ref = x[idx]
        for spec, w in zip(specs, ws):
            s = wf.LayerSpec(len(idx), spec.in_channels, spec.out_channels, spec.height, spec.width, 3, 1, 1)
            ref = O.direct_conv_f64(ref, w, s).astype(np.float32)
        err = O.max_rel_error(y[idx].cpu().numpy(), ref)
        assert err <= len(seg) * TOL, ([layers[i].name for i in seg], err)


@pytest.mark.parametrize("k", range(4))
def test_c4_fft_layer_at_b128(k):
    _check_layer(CONFIGS["c4"][k])


@pytest.mark.parametrize("k", range(12))
def test_c5_layer_at_b256(k):
    variant, _ = _check_layer(CONFIGS["c5"][k])
    assert variant == "ws", variant              # every c5 layer runs the warp-specialised kernel
