"""Suite / report / CLI re-target and layer chaining."""
import json

import numpy as np
import pytest

import paper_1912_02165_b200 as wf
from paper_1912_02165_b200 import cli, suite
from oracle import oracle as O


def _fake_results():
    a = suite.BenchResult(label="l1", engine="fused", tile=6, r=24, workers=148, times_ms=[1.0, 2.0],
                          median_ms=1.5, min_ms=1.0, flops=10, tasks=3, verify="pass", max_rel_err=1e-4,
                          direct_flops=int(3e9), batch=4, t_roof_s=1e-4)
    b = suite.BenchResult(label="l1", engine="three_stage", tile=6, r=24, workers=148, median_ms=3.0,
                          min_ms=2.9, flops=10, direct_flops=int(3e9), batch=4, t_roof_s=1e-4)
    c = suite.BenchResult(label="l2", engine="fused", tile=6, r=24, workers=0, error="boom", verify="error")
    return [a, b, c]


def test_report_formats_share_values():
    res = _fake_results()
    rows = json.loads(suite.emit_report(res, "json"))
    assert [r["engine"] for r in rows] == ["fused", "three_stage", "fused"]
    assert rows[0]["tflops"] == 2.0 and rows[0]["roofline_frac"] == pytest.approx(0.0667, abs=1e-4)
    assert rows[2]["error"] == "boom" and rows[2]["verify"] == "error"
    csv_text = suite.emit_report(res, "csv")
    assert csv_text.splitlines()[0].split(",") == suite.CSV_COLUMNS
    table = suite.emit_report(res, "table")
    assert "2.00x" in table and "error: boom" in table
    with pytest.raises(wf.InvalidParameterError):
        suite.emit_report(res, "xml")
    with pytest.raises(wf.InvalidParameterError):
        suite.emit_report([], "csv")


def test_builtin_suites_and_roofline():
    assert [l for l, _ in suite.builtin_suite("resnet")][0] == "resnet_64ch_56"
    assert len(suite.builtin_suite("vgg16")) == 13 and len(suite.builtin_suite("sweep")) == 12
    with pytest.raises(wf.InvalidParameterError):
        suite.builtin_suite("nope")
    spec = wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1)
    t = suite.roofline_seconds(spec, 6, peaks={"hbm_gbs": 6545.3, "bf16_tflops": 1657.2})
    assert t == pytest.approx(103350272 / 6545.3e9, rel=1e-9)      # c2 is HBM-bound


def test_cli_parser_and_dump_basis(capsys):
    assert cli.main(["dump-basis", "--tile", "4"]) == 0
    out = capsys.readouterr().out
    assert "tile T=4" in out and "[1, 1, 1, 0]" in out
    args = cli.build_parser().parse_args(["bench", "--suite", "resnet", "--engines", "fused", "--transform", "fft"])
    assert args.suite == "resnet" and args.transform == "fft"


def test_layer_stack_rejects_mismatched_layers():
    a = wf.LayerSpec(1, 8, 16, 10, 10, 3, 1, 1)
    b = wf.LayerSpec(1, 8, 8, 10, 10, 3, 1, 1)          # expects 8 channels, gets 16
    with pytest.raises(wf.ShapeMismatchError):
        wf.LayerStack([a, b], [None, None], wf.EngineConfig())


@pytest.mark.gpu
def test_layer_stack_matches_layer_by_layer(cuda_dev):
    import torch
    specs = [wf.LayerSpec(2, 8, 32, 30, 30, 3, 1, 1), wf.LayerSpec(2, 32, 32, 30, 30, 3, 1, 1),
             wf.LayerSpec(2, 32, 16, 30, 30, 3, 1, 1)]
    cfgs = [wf.EngineConfig(kind="fused", tile=6, device=cuda_dev),
            wf.EngineConfig(kind="three_stage", tile=4, device=cuda_dev),
            wf.EngineConfig(kind="fused", transform="fft", tile=16, device=cuda_dev)]
    packs = []
    for i, (s, c) in enumerate(zip(specs, cfgs)):
        w = wf.new_tensor(s.kernel_dims(), seed=10 + i)
        basis = wf.make_fft_basis() if c.transform == "fft" else wf.make_basis(c.tile)
        packs.append(wf.transform_kernels(w, basis))
    x = wf.new_tensor(specs[0].input_dims(), seed=3)
    stack = wf.LayerStack(specs, packs, cfgs)
    y = stack(torch.from_numpy(x.data).to(cuda_dev)).cpu().numpy()
    ref = x
    for s, p, c in zip(specs, packs, cfgs):
        ref, _ = wf.run_engine(c.kind, ref, p, s, c)
    assert np.array_equal(y, ref.data)


@pytest.mark.gpu
def test_run_suite_small_layer_verifies(cuda_dev):
    entries = [("small", wf.LayerSpec(2, 16, 16, 20, 20, 3, 1, 1))]
    res = suite.run_suite(entries, ["fused", "three_stage", "direct"], tile=6, reps=2, warmup=1, verify=True,
                          device=cuda_dev)
    assert all(r.error is None and r.verify == "pass" for r in res), [(r.error, r.verify) for r in res]
    rows = json.loads(suite.emit_report(res, "json"))
    assert all(r["tflops"] > 0 for r in rows)


def test_reference_planner_restatement_matches_published_example():
    # The reference README's planner example (skylakex-like model, C = C' = 64,
    # T = 7): r_lower 20, r_upper 40, predicted utilization 0.457.
    from paper_1912_02165_b200 import roofline
    m = roofline.MachineModel.from_dict({"name": "skylakex-like", "peak_flops": 3.5e12,
                                         "mem_bandwidth_bytes_per_s": 100e9, "l3_bandwidth_bytes_per_s": 350e9,
                                         "l2_bytes_per_core": 1048576, "l3_bytes": 33554432, "cores": 28})
    rep = roofline.plan(wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1), 7, m)
    assert (rep.r_lower, rep.r_upper, rep.chosen_r, rep.feasible) == (20, 40, 40, True)
    assert round(rep.utilization_overall, 3) == 0.457 and rep.l3_fits
    with pytest.raises(wf.MachineModelError):
        roofline.MachineModel.from_dict({"name": "x"})


def test_b200_planner_levels():
    from paper_1912_02165_b200 import roofline
    mach = roofline.B200Model.from_file(roofline.sample_model_path("b200"))
    c2 = roofline.plan_b200(wf.LayerSpec(64, 64, 64, 56, 56, 3, 1, 1), 6, mach)
    assert c2.n_tile == 12544 and c2.blocks == 98
    assert c2.bytes["hbm_fused"] == 103350272                     # Q_fused of SURVEY.md 8(d)
    assert c2.bytes["hbm_three"] == 103350272 + 8 * 36 * 12544 * 128
    assert c2.predicted_winner == "fused" and "persistent" in c2.fused_variant
    assert c2.r_upper < 128 <= c2.r_lower + 64                     # a 128-tile block does not fit one SM
    fft = roofline.plan_b200(wf.LayerSpec(128, 64, 64, 56, 56, 3, 1, 1), 16, mach, transform="fft")
    assert fft.n_tile == 2048 and "waves" in fft.fused_variant
    assert "predicted winner" in c2.format()


@pytest.mark.gpu
def test_host_pipeline_matches_single_call(cuda_dev):
    import torch
    spec = wf.LayerSpec(10, 32, 48, 28, 28, 3, 1, 1)
    w = wf.new_tensor(spec.kernel_dims(), seed=2)
    pack = wf.transform_kernels(w, wf.make_basis(6))
    x = wf.new_tensor(spec.input_dims(), seed=1)
    cfg = wf.EngineConfig(kind="fused", tile=6, device=cuda_dev)
    ref = wf.LayerPlan(spec, pack, cfg)(torch.from_numpy(x.data).to(cuda_dev)).cpu().numpy()
    x_host = torch.from_numpy(x.data).pin_memory()
    y_host = torch.empty(spec.output_dims(), dtype=torch.float32).pin_memory()
    for chunks in (1, 3, 4):
        y_host.zero_()
        wf.HostPipeline(spec, pack, cfg, chunks=chunks)(x_host, y_host)
        assert np.array_equal(y_host.numpy(), ref), chunks


@pytest.mark.gpu
def test_host_pipeline_streaming_submit_wait(cuda_dev):
    """submit() / wait(): calls queued back to back over two staging sets
    (call k + 1 uploads while call k downloads) give, for every call, bitwise
    the single-call result -- different inputs per call, so a staging set
    reused too early would show."""
    import torch
    spec = wf.LayerSpec(6, 64, 64, 24, 24, 3, 1, 1)
    w = wf.new_tensor(spec.kernel_dims(), seed=4)
    pack = wf.transform_kernels(w, wf.make_basis(6))
    cfg = wf.EngineConfig(kind="fused", tile=6, device=cuda_dev)
    plan = wf.LayerPlan(spec, pack, cfg)
    xs = [wf.new_tensor(spec.input_dims(), seed=10 + i).data for i in range(5)]
    refs = [plan(torch.from_numpy(x).to(cuda_dev)).cpu().numpy() for x in xs]
    x_hosts = [torch.from_numpy(x).pin_memory() for x in xs]
    y_hosts = [torch.zeros(spec.output_dims(), dtype=torch.float32).pin_memory() for _ in xs]
    for chunks, depth in ((1, 2), (3, 2), (2, 3), (1, 1)):
        for y in y_hosts:
            y.zero_()
        pipe = wf.HostPipeline(spec, pack, cfg, chunks=chunks, graph=False, depth=depth)
        for xh, yh in zip(x_hosts, y_hosts):
            pipe.submit(xh, yh)
        pipe.wait()
        for i, (yh, ref) in enumerate(zip(y_hosts, refs)):
            assert np.array_equal(yh.numpy(), ref), (chunks, depth, i)
    with pytest.raises(wf.InvalidParameterError):
        wf.HostPipeline(spec, pack, cfg, depth=0)


def test_b200_model_fitted_to_measured_layers():
    """The B200 planner's rates are fitted to measured layer times (the
    warp-specialised fused kernel and the three-stage engine, bench.py
    per_config rows shipped in machines/b200_measured.json): the fit
    reproduces the measurements within ~20% RMS (log) and predicts the
    measured fused / three-stage winner of every layer, including the c5
    crossover sweep."""
    from paper_1912_02165_b200 import roofline
    rows = roofline.measured_layers()
    fit = roofline.fit_b200(rows)
    assert fit.samples == len(rows) >= 12 and fit.rms_log_error < 0.3
    for r in rows:
        want = "fused" if r["fused_s"] < r["three_s"] else "three_stage"
        assert fit.winner(r["layer"], r["tile"]) == want, r["name"]
    shipped = roofline.B200Fit.from_file(roofline.sample_model_path("b200_fit"))
    assert abs(shipped.l2_rate / fit.l2_rate - 1) < 0.05
    rep = roofline.plan_b200(wf.LayerSpec(256, 16, 16, 28, 28, 3, 1, 1), 8)
    assert rep.fitted and rep.predicted_winner == "fused" and "fitted" in rep.format()
