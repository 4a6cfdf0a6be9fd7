"""Host-side API: types, exact bases, tiling, layouts, configs, errors.

Known-answer values follow the reference's own tests (pkg/tests/
test_basis.py, test_tiling.py, test_engines.py, test_tensor.py) and the
golden fixtures generated from the reference.
"""
from fractions import Fraction as F

import numpy as np
import pytest

import paper_1912_02165_b200 as wf
from paper_1912_02165_b200 import engines as eng


# ------------------------------------------------------------------ basis
def test_basis_exact_matrices_match_reference(golden_basis):
    for key, ref in golden_basis.items():
        t, k = (int(v) for v in key[1:].split("_K"))
        b = wf.make_basis(t, k)
        assert [[str(v) for v in r] for r in b.at_exact] == ref["at"], key
        assert [[str(v) for v in r] for r in b.bt_exact] == ref["bt"], key
        assert [[str(v) for v in r] for r in b.g_exact] == ref["g"], key
        assert [str(p) for p in b.points] == ref["points"], key
        if ref["dump"] is not None:
            assert b.dump() == ref["dump"]


def test_f23_pinned_matrices():
    b = wf.make_basis(4, 3, points=(0, 1, -1))
    assert b.out == 2
    assert b.g_exact == ((F(1), F(0), F(0)), (F(1, 2), F(1, 2), F(1, 2)), (F(1, 2), F(-1, 2), F(1, 2)),
                         (F(0), F(0), F(1)))
    assert b.bt_exact == ((F(1), F(0), F(-1), F(0)), (F(0), F(1), F(1), F(0)), (F(0), F(-1), F(1), F(0)),
                          (F(0), F(1), F(0), F(-1)))
    assert b.at_exact == ((F(1), F(1), F(1), F(0)), (F(0), F(1), F(-1), F(-1)))


def _identity_violations(b):
    t, k, m = b.tile, b.kernel, b.out
    bad = 0
    for i in range(t):
        for j in range(t):
            for a in range(k):
                for c in range(k):
                    qa = [sum(b.at_exact[r][p] * b.bt_exact[p][i] * b.g_exact[p][a] for p in range(t))
                          for r in range(m)]
                    qb = [sum(b.at_exact[r][p] * b.bt_exact[p][j] * b.g_exact[p][c] for p in range(t))
                          for r in range(m)]
                    for r in range(m):
                        for s in range(m):
                            want = 1 if (r == i - a and s == j - c) else 0
                            if qa[r] * qb[s] != want:
                                bad += 1
    return bad


@pytest.mark.parametrize("t", range(4, 9))
def test_basis_exact_identity(t):
    assert _identity_violations(wf.make_basis(t, 3)) == 0


def test_basis_validation():
    with pytest.raises(wf.InvalidParameterError):
        wf.make_basis(3, 3)
    with pytest.raises(wf.InvalidParameterError):
        wf.make_basis(9, 3)
    with pytest.raises(wf.InvalidParameterError):
        wf.make_basis(7, 3, points=(0, 1, -1))
    with pytest.raises(wf.BasisConstructionError):
        wf.make_basis(4, 3, points=(0, 1, 1))
    with pytest.raises(wf.BasisConstructionError):
        wf.make_basis(4, 3, points=(0.5, 1, -1))
    with pytest.raises(wf.InvalidParameterError):
        wf.default_points(9)
    assert wf.default_points(8)[-1] == F(-1, 2)


def test_f32_views_readonly():
    for t in range(4, 9):
        b = wf.make_basis(t)
        assert b.at32.dtype == np.float32 and not b.at32.flags.writeable
        assert np.array_equal(b.at32, b.at.astype(np.float32))


def test_generated_kernel_tables_match_basis():
    import re
    import os
    path = os.path.join(os.path.dirname(wf.__file__), "csrc", "basis_tables.cuh")
    text = open(path).read()
    for t in range(4, 9):
        b = wf.make_basis(t)
        for name, mat in (("bt", b.bt32), ("at", b.at32)):
            body = text.split(f"constexpr float {name}<{t}>(int r, int q) {{")[1].split("default:")[0]
            cases = {int(k): float(v.rstrip("f")) for k, v in re.findall(r"case (\d+): return ([-0-9.e]+f);", body)}
            cols = mat.shape[1]
            for r in range(mat.shape[0]):
                for q in range(cols):
                    assert cases.get(r * cols + q, 0.0) == float(mat[r, q])


# ------------------------------------------------------------------ tensors
def test_layer_spec_and_dims():
    s = wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1)
    assert wf.output_dims(s) == (56, 56)
    assert wf.output_tensor_dims(s) == (64, 64, 56, 56)
    assert wf.output_dims(wf.LayerSpec(1, 1, 1, 7, 7, 3)) == (5, 5)
    with pytest.raises(wf.InvalidDimensionError):
        wf.LayerSpec(0, 1, 1, 5, 5)
    with pytest.raises(wf.InvalidDimensionError):
        wf.LayerSpec(1, 1, 1, 1, 1, 3, 0, 0)
    with pytest.raises(wf.InvalidDimensionError):
        wf.LayerSpec(1, 1, 1, 5, 5, 3, -1, 0)


def test_new_tensor_seed_matches_reference_rng(golden_cases):
    c = next(c for c in golden_cases if c["name"] == "t4_r3")
    spec = wf.LayerSpec(*c["dims"])
    assert np.array_equal(wf.new_tensor(spec.input_dims(), seed=c["seed_x"]).data, c["x"])
    t = wf.new_tensor((2, 3, 4, 5), fill=1)
    assert t.data.sum() == 120 and t.data.ctypes.data % 64 == 0
    with pytest.raises(wf.InvalidDimensionError):
        wf.new_tensor((1, 0, 2, 2))
    assert t.flat_index(1, 2, 3, 4) == 119


# ------------------------------------------------------------------ tiling
def test_tile_plan_counts():
    pl = wf.tile_plan(wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1), 7)
    assert (pl.out, pl.tiles_y, pl.tiles_x, pl.n_tile) == (5, 12, 12, 9216)
    vgg = wf.tile_plan(wf.LayerSpec(64, 64, 64, 224, 224, 3, 1, 1), 7)
    assert vgg.n_tile == 129600
    c2 = wf.tile_plan(wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1), 6)
    assert c2.n_tile == 12544
    with pytest.raises(wf.InvalidParameterError):
        wf.tile_plan(wf.LayerSpec(1, 1, 1, 5, 5), 3)


def test_tile_coords_round_trip_and_origins():
    pl = wf.tile_plan(wf.LayerSpec(3, 2, 2, 17, 23, 3, 1, 0), 6)
    for i in range(pl.n_tile):
        c = pl.coord(i)
        assert pl.encode(c.batch, c.tile_row, c.tile_col) == i
    big = wf.tile_plan(wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1), 7)
    assert big.input_origin(big.coord(0)) == (-1, -1)
    assert big.output_origin(big.coord(big.encode(0, 11, 11))) == (55, 55)


def test_gather_and_scatter_edges():
    spec = wf.LayerSpec(1, 1, 1, 3, 3, 3, 1, 1)
    pl = wf.tile_plan(spec, 4)
    tile = wf.gather_input_tile(wf.new_tensor(spec.input_dims(), fill=1), pl, pl.coord(0), 0)
    assert np.array_equal(tile, np.array([[0, 0, 0, 0], [0, 1, 1, 1], [0, 1, 1, 1], [0, 1, 1, 1]], np.float32))
    spec = wf.LayerSpec(2, 1, 1, 13, 11, 3, 1, 0)
    pl = wf.tile_plan(spec, 5)
    out = wf.new_tensor(spec.output_dims(), fill=-1)
    counts = np.zeros(spec.output_dims(), np.int32)
    for i in range(pl.n_tile):
        c = pl.coord(i)
        wf.scatter_output_tile(out, pl, c, 0, np.full((pl.out, pl.out), float(i), np.float32))
        oy, ox = pl.output_origin(c)
        counts[c.batch, 0, oy:oy + pl.out, ox:ox + pl.out] += 1
    assert (counts == 1).all() and (out.data >= 0).all()


# ------------------------------------------------------------ engine config
def test_engine_config_validation():
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(kind="blocked")
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(kind="fused", tile=3)
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(kind="fused", tile=9)
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(kind="fused", r=0)
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(kind="fused", workers=-1)
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(kind="fused", precision="fp8")
    with pytest.raises(wf.InvalidParameterError):
        wf.EngineConfig(kind="fused", transform="fft", tile=6)
    wf.EngineConfig(kind="direct", tile=3)
    cfg = wf.EngineConfig(kind="fused", workers=6)
    assert cfg.resolved_workers() == 6 and cfg.resolved_workers(cap=2) == 2
    assert wf.EngineConfig(kind="fused", transform="fft", tile=16).tile == 16


def test_run_engine_rejects_unknown_kind():
    spec = wf.LayerSpec(1, 2, 2, 6, 6, 3, 1, 1)
    with pytest.raises(wf.InvalidParameterError):
        wf.run_engine("winograd", wf.new_tensor(spec.input_dims()), wf.new_tensor(spec.kernel_dims()), spec)


# ----------------------------------------------------------- buffer layout
def test_buffer_layout_pinned_examples():
    lo = wf.buffer_layout(2, 4, 4, 2)
    assert (lo.s_l, lo.s_r, lo.capacity) == (32, 32, 160)
    assert lo.result_offsets == (0, 32, 64, 96) and lo.left_offsets == (32, 64, 96, 128)
    assert lo.left_offset(1) == 32 and lo.result_offset(1) == 0
    cap, lofs, rofs = lo
    assert cap == 160
    lo = wf.buffer_layout(2, 3, 5, 2)
    assert (lo.s_l, lo.s_r, lo.capacity) == (24, 40, 184)
    assert wf.buffer_layout(24, 64, 64, 7).capacity == 307200
    with pytest.raises(wf.InvalidParameterError):
        wf.buffer_layout(0, 4, 4, 4)


def test_buffer_layout_no_overlap_grid():
    for r in (1, 7, 64):
        for c in (8, 64, 512):
            for cp in (8, 64, 512):
                for t in range(4, 9):
                    lo = wf.buffer_layout(r, c, cp, t)
                    assert lo.capacity == t * t * lo.s_max + lo.s_min
                    assert all(lo.result_offsets[p] + lo.s_r <= lo.left_offsets[p] for p in range(t * t))


def test_shared_buffer_views_alias():
    lo = wf.buffer_layout(3, 8, 4, 4)
    buf = wf.SharedBuffer(lo)
    assert buf.flat.ctypes.data % 64 == 0
    assert buf.left.shape == (16, 3, 8) and buf.result.shape == (16, 3, 4)
    assert np.shares_memory(buf.left, buf.result)


# ------------------------------------------------------------- kernel packs
def test_host_pack_bitwise_vs_reference(golden_cases):
    for c in golden_cases:
        pack = wf.transform_kernels(wf.Tensor4D(c["w"]), wf.make_basis(c["tile"]))
        assert np.array_equal(pack.data, c["pack"]), c["name"]
        assert not pack.data.flags.writeable and pack.data.ctypes.data % 64 == 0
        assert pack.nbytes == c["pack"].nbytes


def test_pack_metadata_and_errors():
    pack = wf.transform_kernels(wf.new_tensor((5, 3, 3, 3)), wf.make_basis(6))
    assert pack.data.shape == (36, 3, 5)
    assert (pack.tile, pack.kernel_side, pack.c_in, pack.c_out) == (6, 3, 3, 5)
    with pytest.raises(wf.ShapeMismatchError):
        wf.transform_kernels(wf.new_tensor((1, 1, 5, 5)), wf.make_basis(7))


def test_multiply_flops():
    assert wf.multiply_flops(3, 5, 2, 4) == 2 * 3 * 5 * 2 * 16


def test_errors_hierarchy():
    e = wf.IntermediateAllocationError(7225344, "staged")
    assert isinstance(e, MemoryError) and isinstance(e, wf.WinofuseError) and "7225344" in str(e)
    assert issubclass(wf.UnsupportedConfigError, wf.InvalidParameterError)
    assert issubclass(wf.ShapeMismatchError, ValueError)


def test_fused_rejects_raw_kernels_before_touching_the_gpu():
    spec = wf.LayerSpec(1, 2, 2, 6, 6, 3, 1, 1)
    with pytest.raises(wf.ShapeMismatchError):
        wf.conv_fused(wf.new_tensor(spec.input_dims()), wf.new_tensor(spec.kernel_dims()), spec,
                      wf.EngineConfig(kind="fused", tile=4))


def test_pack_must_match_config_before_gpu():
    spec = wf.LayerSpec(1, 2, 2, 6, 6, 3, 1, 1)
    pack6 = wf.transform_kernels(wf.new_tensor(spec.kernel_dims()), wf.make_basis(6))
    with pytest.raises(wf.ShapeMismatchError):
        wf.conv_fused(wf.new_tensor(spec.input_dims()), pack6, spec, wf.EngineConfig(kind="fused", tile=7))
