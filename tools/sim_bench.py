"""Device-resident backward-Euler simulation vs the reference's run_simulation
(SURVEY.md §8f rank 3).  python tools/sim_bench.py [cells] [steps] [dt] [tol]
Defaults: the converging regime (h = 1 s, tol 1e-10); at the paper's h = 120 s
/ tol 1e-30 -- and after a few steps even here -- the synthetic trajectory
blows up (Newton never converges, half the states clip) and
Jacobi-BiCGSTAB's LU fallback meets an exactly singular Newton matrix or a state
goes non-finite, as in the reference; the default is one step.
Prints one JSON line: steps/s and cell-steps/s of bc_simulate (Block-cells(1),
both algorithms) and of the reference's own run_simulation (oracle/_ref,
Block-cells(1) BiCG, all host threads) on a bounded cell sample, with the
per-step Newton iterations and solver iterations of both."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402,F401

from paper_2405_17363_b200 import Algo, Mechanism, Strategy, StrategyConfig  # noqa: E402
from paper_2405_17363_b200.simulate import LinearSolverChoice, SimulationConfig, run_simulation  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dt = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-10
mech = Mechanism(156, 468, 0)
out = {"workload": f"M156, {cells} cells, Realistic, {steps} steps of h = {dt:g} s, tol {tol:g}, max_iter 1000, "
                   "newton_rtol 1e-10, <= 10 Newton iterations"}
for algo in (Algo.BICGSTAB_JACOBI, Algo.BICG):
    cfg = SimulationConfig(cells=cells, mode=1, steps=steps, dt_seconds=dt, tol=tol,
                           solver=LinearSolverChoice(False, StrategyConfig(Strategy.BlockCells, 1), algo))
    run_simulation(mech, SimulationConfig(cells=cells, mode=1, steps=1, dt_seconds=dt, tol=tol,
                                          solver=cfg.solver, max_newton_iterations=1))  # plans, warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        res = run_simulation(mech, cfg)
    except Exception as e:  # SolverAbort / SingularMatrix: the synthetic trajectory blows up
        out[algo.name.lower()] = {"error": f"{type(e).__name__}: {e}"}
        continue
    el = time.perf_counter() - t0
    out[algo.name.lower()] = {"seconds": el, "cell_steps_per_s": cells * steps / el,
                              "solve_seconds": sum(s.wall_time_ns for s in res.per_step) / 1e9,
                              "newton_iterations": [s.newton_iterations for s in res.per_step],
                              "iterations_sum": [s.iterations_sum for s in res.per_step],
                              "clip_events": [s.clip_events for s in res.per_step]}
import oracle_ffi as of  # noqa: E402
if of.have_ref():
    sample = min(cells, 2 * (os.cpu_count() or 1))
    t0 = time.perf_counter()
    st, r = of.ref_run_simulation(156, 468, 0, sample, 1, 1, dt, tol, 1000, 2, 1, False,
                                  workers=os.cpu_count() or 1)
    el = time.perf_counter() - t0
    out["reference_bicg"] = {"cells_sample": sample, "steps": 1, "seconds": el, "cell_steps_per_s": sample / el,
                             "threads": os.cpu_count(), "newton_iterations": [s["newton_iterations"] for s in r.per_step]}
print(json.dumps(out))
