"""The CPU oracle pinned against the reference's own outputs (tests/golden).

The oracle (oracle/winofuse_oracle.c) restates the reference kernels in C;
here it must reproduce the reference's fused, three-stage and direct
engines BIT FOR BIT on every golden case, for any worker count -- which is
what makes it a valid checker for the GPU parity tests.
"""
import numpy as np
import pytest

from oracle import oracle as O
import paper_1912_02165_b200 as wf


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_fused_bitwise_vs_reference(golden_cases, threads):
    for c in golden_cases:
        spec = wf.LayerSpec(*c["dims"])
        got = O.conv_fused(c["x"], c["pack"], spec, c["tile"], c["r"], threads=threads)
        assert np.array_equal(got, c["fused"]), c["name"]


def test_oracle_three_stage_bitwise_vs_reference(golden_cases):
    for c in golden_cases:
        spec = wf.LayerSpec(*c["dims"])
        got = O.conv_three_stage(c["x"], c["pack"], spec, c["tile"], threads=2)
        assert np.array_equal(got, c["three_stage"]), c["name"]


def test_oracle_direct_bitwise_vs_reference(golden_cases):
    for c in golden_cases:
        spec = wf.LayerSpec(*c["dims"])
        assert np.array_equal(O.direct_conv_f32(c["x"], c["w"], spec), c["direct"]), c["name"]


def test_oracle_pack_bitwise_vs_reference(golden_cases):
    for c in golden_cases:
        assert np.array_equal(O.transform_kernels(c["w"], c["tile"]), c["pack"]), c["name"]


def test_f64_direct_oracle_vs_reference_direct(golden_cases):
    for c in golden_cases:
        spec = wf.LayerSpec(*c["dims"])
        assert O.max_rel_error(c["direct"], O.direct_conv_f64(c["x"], c["w"], spec)) <= 1e-6, c["name"]


def test_all_ones_pinned_output(golden_cases):
    c = next(c for c in golden_cases if c["name"] == "ones_3x3")
    want = np.array([[4, 6, 4], [6, 9, 6], [4, 6, 4]], np.float32)
    assert np.array_equal(c["direct"][0, 0], want)
    assert np.array_equal(O.direct_conv_f32(c["x"], c["w"], wf.LayerSpec(*c["dims"]))[0, 0], want)


def test_reference_fused_tolerance_on_golden(golden_cases):
    # the reference's own acceptance bar, max_rel_error <= 1e-4 vs direct
    for c in golden_cases:
        assert O.max_rel_error(c["fused"], c["direct"]) <= 1e-4, c["name"]


def test_stage_functions_match_fused(golden_cases):
    c = next(c for c in golden_cases if c["name"] == "t6_short_last_task")
    spec = wf.LayerSpec(*c["dims"])
    t = c["tile"]
    n = wf.tile_plan(spec, t).n_tile
    left = O.forward_tiles(c["x"], spec, t, 0, n, n)
    res = O.multiply_positions(left, c["pack"], n)
    out = O.inverse_tiles(res, spec, t, 0, n)
    assert np.array_equal(out, c["three_stage"])
