"""The bench layer (experiment.py) against the
reference's own bench.cpp / format.cpp / exec_model.cpp (oracle/_ref):
results.csv text byte for byte, std::to_chars formatting, summary.json read
back by summary_stats_from_json and re-emitted identically, and the analytic
kernel plan / occupancy / memory census.  The GPU test runs a small
experiment end to end through the device simulation."""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle_ffi as of
from paper_2405_17363_b200 import Strategy, StrategyConfig
from paper_2405_17363_b200 import experiment as ex

needs_ref = pytest.mark.skipif(not of.have_ref(), reason="oracle/_ref (the compiled reference) not built")
KIND = {Strategy.OneCell: 0, Strategy.MultiCells: 1, Strategy.BlockCells: 2}


def ref_format(v):
    buf = C.create_string_buffer(64)
    assert of.ref().ref_format_double(v, buf) == 0
    return buf.value.decode()


@needs_ref
def test_format_double_is_to_chars():
    rng = np.random.default_rng(0)
    vals = [0.0, -0.0, 1.0, 0.5, 0.1, 1 / 3, 120.0, 1e-30, 1e22, 1e21, 1e16, 1e15, 123456.0, 100000.0, 1e5 + 1,
            5e-324, 1.7976931348623157e308, 2.2250738585072014e-308, 6.564102564102564, 1e-4, 1.5e-5, 0.001,
            12345678901234567890.0, 9.999999999999999e22, 1234.5, -2.5e-7, math.inf, -math.inf]
    vals += list(rng.standard_normal(200) * 10.0 ** rng.integers(-40, 40, 200))
    vals += [float(x) for x in rng.integers(0, 10 ** 9, 50)]
    for v in vals:
        assert ex.format_double(float(v)) == ref_format(float(v)), v


@needs_ref
def test_csv_is_the_reference_text():
    rng = np.random.default_rng(1)
    rows = []
    for i in range(40):
        rows.append(ex.StepRecord(i % 7, ["one-cell", "block-cells", "multi-cells"][i % 3], int(rng.integers(1, 10 ** 6)),
                                  156, float(rng.choice([1.0, 6.0, 6.564102564102564, 3.0])),
                                  int(rng.integers(0, 10 ** 7)), int(rng.integers(0, 10 ** 9)),
                                  int(rng.integers(0, 10 ** 12)), float(rng.standard_normal() * 10.0 ** rng.integers(-30, 30)),
                                  int(rng.integers(0, 300)), int(rng.integers(0, 5000))))
    cols = lambda f, t: np.array([getattr(r, f) for r in rows], t)  # noqa: E731
    names = b"".join(r.strategy.encode() + b"\0" for r in rows)
    arrs = [cols("step", np.int64), cols("cells", np.int64), cols("species", np.int64),
            cols("cells_per_block", np.float64), cols("iterations_effective", np.int64),
            cols("iterations_sum", np.int64), cols("wall_ns", np.int64), cols("max_residual_rms", np.float64),
            cols("breakdown_fallbacks", np.int64), cols("clip_events", np.int64)]
    st = of.ref().ref_to_csv(len(rows), of.ptr(arrs[0]), names, *[of.ptr(a) for a in arrs[1:]])
    assert st == 0
    want = of.ref().ref_last_text().decode()
    assert ex.to_csv(rows) == want
    assert ex.parse_csv(want) == rows


@needs_ref
@pytest.mark.parametrize("kind,cells,species,k,mtpb", [
    (Strategy.OneCell, 1000, 156, 0, 1024), (Strategy.MultiCells, 1000, 156, 0, 1024),
    (Strategy.BlockCells, 1000, 156, 0, 1024), (Strategy.BlockCells, 1000, 156, 1, 1024),
    (Strategy.BlockCells, 100001, 156, 4, 1024), (Strategy.BlockCells, 7, 312, 0, 1024),
    (Strategy.MultiCells, 3, 1024, 0, 1024), (Strategy.OneCell, 10, 1000, 0, 1024),
    (Strategy.BlockCells, 11, 33, 0, 512)])
def test_kernel_plan_model_is_the_reference(kind, cells, species, k, mtpb):
    import json
    assert of.ref().ref_plan_json(KIND[kind], cells, species, k, mtpb) == 0
    text = of.ref().ref_last_text().decode()
    plan_json, tail = text.rsplit("\n", 1)
    dev = ex.DeviceSpec(max_threads_per_block=mtpb, max_threads_per_sm=max(2048, mtpb))
    plan = ex.plan_kernel(kind, cells, species, dev, k or None)
    assert ex._dump(plan.to_json_obj()) == plan_json
    occ, exceeded = ex.occupancy_estimate(plan, dev)
    o, e, mp, ma = tail.split()
    assert ex.format_double(occ) == o and int(exceeded) == int(e)
    assert ex.memory_estimate(kind, cells, species, 9, dev, k or None) == int(mp)
    assert ex.memory_estimate(kind, cells, species, 6, dev, k or None) == int(ma)
    assert json.loads(plan_json)["strategy"] == ex.STRATEGY_NAMES[kind]


def _synthetic_stats(cfg):
    rng = np.random.default_rng(2)
    out = []
    for i, sc in enumerate(cfg.strategies):
        k = sc.cells_per_block if sc.kind == Strategy.BlockCells else None
        plan = ex.plan_kernel(sc.kind, cfg.cells, cfg.species, cfg.device, k)
        occ, exc = ex.occupancy_estimate(plan, cfg.device)
        out.append(ex.StrategyStats(
            config=sc, plan=plan, occupancy=occ, occupancy_shared_mem_exceeded=exc,
            memory_bytes_paper_census=ex.memory_estimate(sc.kind, cfg.cells, cfg.species, 9, cfg.device, k),
            memory_bytes_actual_census=ex.memory_estimate(sc.kind, cfg.cells, cfg.species, 6, cfg.device, k),
            iterations_effective=ex.mean_std(rng.integers(1, 1000, 9)), wall_ns=ex.mean_std(rng.integers(1, 10 ** 9, 9)),
            speedup_vs_baseline=None if i == 0 else float(rng.uniform(0.1, 50)),
            iteration_reduction_vs_block1=None if i == 1 else ex.mean_std(rng.uniform(0.5, 2.0, 9))))
    return out


def _roundtrip(cfg, text):
    kinds = np.array([KIND[s.kind] for s in cfg.strategies], np.int32)
    ks = np.array([s.cells_per_block or 0 for s in cfg.strategies], np.int64)
    st = of.ref().ref_summary_roundtrip(text.encode(), cfg.cells, cfg.species, cfg.steps, cfg.dt_seconds, cfg.mode,
                                        len(kinds), of.ptr(kinds), of.ptr(ks), cfg.tol, cfg.max_iter, cfg.seed,
                                        cfg.worker_count, cfg.output_path.encode())
    assert st == 0
    return of.ref().ref_last_text().decode()


@needs_ref
def test_summary_json_round_trips_through_the_reference():
    cfg = ex.ExperimentConfig(cells=1000, species=156, steps=9, strategies=[
        StrategyConfig(Strategy.OneCell), StrategyConfig(Strategy.BlockCells, 1), StrategyConfig(Strategy.BlockCells),
        StrategyConfig(Strategy.MultiCells), StrategyConfig(Strategy.BlockCells, 4)], output_path="out/run1")
    stats = _synthetic_stats(cfg)
    text = ex.summary_to_json(cfg, stats)
    assert _roundtrip(cfg, text) == text  # read back and re-emitted byte for byte


def test_mean_std_two_pass():
    m = ex.mean_std([3.0, 3.0, 3.0])
    assert m.mean == 3.0 and m.std == 0.0
    m = ex.mean_std([1.0, 2.0, 3.0, 4.0])
    assert m.mean == 2.5 and m.std == math.sqrt(1.25)
    assert ex.mean_std([]) == ex.MeanStd()
    with pytest.raises(ValueError):
        ex.ExperimentConfig(strategies=[]).check()


@pytest.mark.gpu
def test_experiment_on_the_gpu_reads_back_in_the_reference(tmp_path, solver):
    cfg = ex.ExperimentConfig(cells=12, species=24, steps=2, dt_seconds=120.0, max_iter=200, seed=3,
                              strategies=[StrategyConfig(Strategy.OneCell), StrategyConfig(Strategy.BlockCells, 1),
                                          StrategyConfig(Strategy.BlockCells)],
                              output_path=str(tmp_path / "exp"))
    res = ex.run_experiment(cfg)
    ex.write_outputs(cfg, res)
    text = open(os.path.join(cfg.output_path, "results.csv")).read()
    assert ex.parse_csv(text) == res.raw and len(res.raw) == 6
    # one-cell and block-cells(1) solve the same systems: same iterations
    assert [r.iterations_effective for r in res.raw[:2]] == [r.iterations_effective for r in res.raw[2:4]]
    assert res.per_strategy[1].iteration_reduction_vs_block1.mean == 1.0
    np.testing.assert_array_equal(res.final_states_per_strategy[0], res.final_states_per_strategy[1])
    if of.have_ref():
        js = open(os.path.join(cfg.output_path, "summary.json")).read().rstrip("\n")
        import json
        stripped = json.loads(js)
        for s in stripped["strategies"]:
            s.pop("b200", None)
        plain = ex._dump(stripped)
        assert _roundtrip(cfg, js) == plain
        # and the per-step records equal the reference's own simulation
        for i, sc in enumerate(cfg.strategies):
            st, want = of.ref_run_simulation(24, 72, 3, 12, 1, 2, 120.0, 1e-30, 200, KIND[sc.kind],
                                             sc.cells_per_block or 0, False)
            assert st == 0
            for r, w in zip(res.raw[2 * i:2 * i + 2], want.per_step):
                assert (r.iterations_effective, r.iterations_sum, r.breakdown_fallbacks, r.clip_events) == (
                    w["iterations_effective"], w["iterations_sum"], w["breakdown_fallbacks"], w["clip_events"])
                assert of.bits(r.max_residual_rms) == of.bits(w["max_residual_rms"])
