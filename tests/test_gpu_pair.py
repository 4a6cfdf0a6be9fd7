"""CTA-pair position GEMM (csrc/gemm_pair.cu, tcgen05.mma.cta_group::2).

The pair kernel runs the position GEMM of the three-stage path and of the L2
waves whenever C_pad is a multiple of 64 and the launch has an even number
of 128-tile blocks (or at least 7).  Covered here: even and odd block counts
(the odd pair's second CTA re-reads the last block and stores nothing), the
complex-structured FFT-16 pack, both precision modes, and bit-identity with
the single-CTA kernel (same MMA K order per accumulator row), checked in two
subprocesses because the WF_GEMM_PAIR switch is read once per process.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1912_02165_b200 as wf
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _layer(b, c, cp, hw, seed):
    rng = np.random.default_rng(seed)
    spec = wf.LayerSpec(b, c, cp, hw, hw, 3, 1, 1)
    x = rng.standard_normal(spec.input_dims()).astype(np.float32)
    w = (rng.standard_normal(spec.kernel_dims()) * np.sqrt(2.0 / (9 * c))).astype(np.float32)
    return spec, x, w


def _run(kind, x, pack, spec, t, **kw):
    cfg = wf.EngineConfig(kind=kind, tile=t, **kw)
    out, _ = wf.run_engine(kind, wf.Tensor4D(x), pack, spec, cfg)
    return out.data


# (B, C, C', HW): blocks of 128 tiles = ceil(B * tiles / 128)
CASES = [
    (4, 256, 512, 28),   # 196 tiles: 2 blocks (one pair), N chunks 2 x 256
    (18, 64, 256, 28),   # 882 tiles: 7 blocks (odd: the last pair is half idle)
    (6, 128, 192, 56),   # 1176 tiles: 10 blocks, N = 192
]


@pytest.mark.parametrize("b,c,cp,hw", CASES)
@pytest.mark.parametrize("kind", ["three_stage", "fused"])
def test_pair_gemm_layers_vs_fp64(b, c, cp, hw, kind):
    spec, x, w = _layer(b, c, cp, hw, b * 1000 + c + cp)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(6))
    y = _run(kind, x, pack, spec, 6, fused_variant="waves") if kind == "fused" else _run(kind, x, pack, spec, 6)
    assert O.max_rel_error(y, O.direct_conv_f64(x, w, spec)) <= 1e-3


def test_pair_gemm_fft16_vs_fp64():
    # FFT-16 (14 x 14 outputs per tile): 2 x 2 tiles per 28 x 28 image,
    # B = 64 -> 256 tiles = 2 blocks; K = 2 C = 256 (re | im)
    spec, x, w = _layer(64, 128, 256, 28, 7)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis(3))
    y = _run("three_stage", x, pack, spec, 16, transform="fft")
    assert O.max_rel_error(y, O.direct_conv_f64(x, w, spec)) <= 1e-3


_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1912_02165_b200 as wf
rng = np.random.default_rng(3)
spec = wf.LayerSpec(18, 64, 256, 28, 28, 3, 1, 1)
x = rng.standard_normal(spec.input_dims()).astype(np.float32)
w = (rng.standard_normal(spec.kernel_dims()) * 0.05).astype(np.float32)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(6))
out = []
for prec in ("3xbf16", "bf16"):
    cfg = wf.EngineConfig(kind="three_stage", tile=6, precision=prec)
    y, _ = wf.run_engine("three_stage", wf.Tensor4D(x), pack, spec, cfg)
    out.append(np.ascontiguousarray(y.data))
np.save(sys.argv[1], np.stack(out))
"""


def test_pair_gemm_bitwise_equals_single_cta(tmp_path):
    res = {}
    for flag in ("0", "1"):
        path = str(tmp_path / f"y{flag}.npy")
        env = dict(os.environ, WF_GEMM_PAIR=flag)
        subprocess.run([sys.executable, "-c", _CHILD.format(root=ROOT), path], env=env, check=True, timeout=300)
        res[flag] = np.load(path)
    assert np.array_equal(res["0"], res["1"])
