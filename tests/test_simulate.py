"""Device-resident backward-Euler simulation (bc_simulate, SURVEY.md §8f
rank 3) against the reference's own run_simulation (oracle/_ref, BiCG and
the dense-LU path) and against the checkers' restatement of the same loop
(tests/oracle_ffi.py orc_run_simulation, any algorithm).  The bar is
bitwise: final states and every per-step field but wall time.

CPU tests pin the restatement against the reference; GPU tests run the
product path."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_ffi as of
from paper_2405_17363_b200 import Algo, Mechanism, Strategy, StrategyConfig

IDEAL, REALISTIC = 0, 1
STRAT = {Strategy.OneCell: 0, Strategy.MultiCells: 1, Strategy.BlockCells: 2}


def assert_same_run(got_states, got_steps, want):
    np.testing.assert_array_equal(of.bits(got_states), of.bits(want.states))
    assert len(got_steps) == len(want.per_step)
    for g, w in zip(got_steps, want.per_step):
        for f in of.STEP_FIELDS:
            if f == "wall_time_ns":
                continue
            gv = g[f] if isinstance(g, dict) else getattr(g, f)
            if f == "max_residual_rms":
                assert of.bits(gv) == of.bits(w[f]), (f, gv, w[f])
            else:
                assert gv == w[f], (f, gv, w[f])


# --- CPU: the restatement is the reference ----------------------------------

needs_ref = pytest.mark.skipif(not of.have_ref(), reason="oracle/_ref (the compiled reference) not built")


@needs_ref
@pytest.mark.parametrize("strategy,k,direct,mode,dt", [
    (Strategy.BlockCells, 1, False, REALISTIC, 120.0),
    (Strategy.OneCell, 0, False, IDEAL, 120.0),
    (Strategy.BlockCells, 0, False, REALISTIC, 1.0),
    (Strategy.MultiCells, 0, False, REALISTIC, 30.0),
    (None, 0, True, REALISTIC, 120.0),
])
def test_oracle_simulation_is_the_reference(strategy, k, direct, mode, dt):
    mech = Mechanism(24, 72, 3)
    cells, steps = 6, 3
    s = STRAT.get(strategy, 0)
    st, want = of.ref_run_simulation(24, 72, 3, cells, mode, steps, dt, 1e-30, 150, s, k, direct, workers=4)
    assert st == 0
    st, got = of.orc_run_simulation(mech, cells, mode, steps, dt, 1e-30, 150, s, k, 0, direct)
    assert st == 0
    assert_same_run(got.states, got.per_step, want)


@needs_ref
def test_oracle_simulation_abort_is_the_reference():
    mech = Mechanism(16, 48, 1)
    y0 = np.ones((4, 16))
    y0[2, 5] = np.inf
    st, want = of.ref_run_simulation(16, 48, 1, 4, REALISTIC, 2, 120.0, 1e-30, 50, 2, 1, False, states=y0)
    assert st == -9 and want.abort_step == 0
    st, got = of.orc_run_simulation(mech, 4, REALISTIC, 2, 120.0, 1e-30, 50, 2, 1, 0, False, states=y0)
    assert st == -9 and got.abort_step == 0


# --- GPU: bc_simulate ----------------------------------------------------------

def run_device(mech, cells, mode, steps, dt, tol, max_iter, strategy, k, algo, direct, states=None):
    from paper_2405_17363_b200.simulate import LinearSolverChoice, SimulationConfig, run_simulation
    cfg = SimulationConfig(cells=cells, mode=mode, steps=steps, dt_seconds=dt, tol=tol, max_iter=max_iter,
                           solver=LinearSolverChoice(direct, StrategyConfig(strategy or Strategy.OneCell,
                                                                            k or None), algo))
    return run_simulation(mech, cfg, states)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy,k,direct,mode", [
    (Strategy.BlockCells, 1, False, REALISTIC),
    (Strategy.OneCell, 0, False, IDEAL),
    (Strategy.BlockCells, 0, False, REALISTIC),
    (None, 0, True, REALISTIC),
])
def test_device_simulation_matches_reference(solver, strategy, k, direct, mode):
    """M156, 24 cells, 2 steps of h = 120 s, P-regime solver settings."""
    if not of.have_ref():
        pytest.skip("oracle/_ref not built")
    mech = Mechanism(156, 468, 0)
    cells, steps = 24, 2
    s = STRAT.get(strategy, 0)
    st, want = of.ref_run_simulation(156, 468, 0, cells, mode, steps, 120.0, 1e-30, 1000, s, k, direct, workers=8)
    assert st == 0
    res = run_device(mech, cells, mode, steps, 120.0, 1e-30, 1000, strategy, k, Algo.BICG, direct)
    assert_same_run(res.final_states, res.per_step, want)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 0])
def test_device_simulation_bicgstab_matches_oracle(solver, k):
    """Jacobi-BiCGSTAB Newton loop (no reference implementation): against the
    restatement driven by the C oracle."""
    mech = Mechanism(156, 468, 0)
    cells, steps = 16, 2
    st, want = of.orc_run_simulation(mech, cells, REALISTIC, steps, 1.0, 1e-10, 1000, 2, k, 1, False)
    assert st == 0
    res = run_device(mech, cells, REALISTIC, steps, 1.0, 1e-10, 1000, Strategy.BlockCells, k,
                     Algo.BICGSTAB_JACOBI, False)
    assert_same_run(res.final_states, res.per_step, want)


@pytest.mark.gpu
def test_device_simulation_abort_and_trivial_cases(solver):
    from paper_2405_17363_b200.simulate import SolverAbort
    mech = Mechanism(24, 72, 3)
    y0 = np.ones((5, 24))
    y0[3, 7] = np.nan
    with pytest.raises(SolverAbort) as e:
        run_device(mech, 5, REALISTIC, 3, 120.0, 1e-30, 100, Strategy.BlockCells, 1, Algo.BICG, False, states=y0)
    assert e.value.step == 0
    # zero steps: the initial state comes back (test_problem_gen.cpp:314-326)
    y1 = np.random.default_rng(0).uniform(0.5, 2.0, (5, 24))
    r = run_device(mech, 5, REALISTIC, 0, 120.0, 1e-30, 100, Strategy.BlockCells, 1, Algo.BICG, False, states=y1)
    np.testing.assert_array_equal(r.final_states, y1)
    assert r.per_step == []
    # ideal mode keeps every cell bit-identical (test_problem_gen.cpp:328-348)
    r = run_device(mech, 6, IDEAL, 3, 120.0, 1e-30, 100, Strategy.BlockCells, 1, Algo.BICG, False)
    for c in range(1, 6):
        np.testing.assert_array_equal(of.bits(r.final_states[c]), of.bits(r.final_states[0]))
    with pytest.raises(ValueError):
        run_device(mech, 5, REALISTIC, 1, 0.0, 1e-30, 100, Strategy.BlockCells, 1, Algo.BICG, False)


@pytest.mark.gpu
def test_cpp_dropin_device_simulation_equals_reference_loop():
    """tests/cpp/test_simulate_dropin.cpp: the shim's blockcells::b200::run_simulation
    (bc_simulate) against the reference's run_simulation (simulate.cpp) over the
    shim's GPU run_strategy, bit for bit, BiCG on every strategy and the LU path,
    Jacobi-BiCGSTAB, and the same errors."""
    import os
    import re
    import subprocess
    binary = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "bin", "sim_dropin")
    if not os.path.exists(binary):
        pytest.skip("tests/cpp binaries not built (needs /root/reference at build time)")
    r = subprocess.run([binary], capture_output=True, text=True, timeout=900)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed; checks: (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-2000:]
    assert int(m.group(3)) == 0 and int(m.group(5)) == 0, r.stdout[-3000:]
    assert int(m.group(1)) == 3
