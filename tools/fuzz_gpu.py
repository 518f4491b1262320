"""Randomised GPU-vs-oracle fuzzing beyond the committed tests (run under gpurun):
    python tools/fuzz_gpu.py [seconds] [seed]
Each case draws a mechanism (generated, or a random diagonally dominant
pattern), a batch size, a strategy (Block-cells(k) / (N), One-cell, Multi-cells,
thread-per-cell), an algorithm and solver settings, a kernel policy (latency
mode forced on / off / default) and a front end (one Solver, or a DeviceSet
listing GPU 0 two or three times), solves it through the public API and
compares x, iterations, residuals and flags bit for bit with the C oracle
(tests/oracle_ffi.py).  Prints one line per case and a summary;
exit status 1 on any mismatch."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_ffi as of  # noqa: E402
from fixtures import random_batch  # noqa: E402
from paper_2405_17363_b200 import (Algo, BatchedSystem, DeviceSet, DeviceSpec, Mechanism, Solver,  # noqa: E402
                                   Strategy, StrategyConfig)

STRAT_ORC = {Strategy.OneCell: 0, Strategy.MultiCells: 1, Strategy.BlockCells: 2, Strategy.ThreadPerCell: 0}


def case(rng):
    if rng.random() < 0.25:  # breakdowns, signed zeros, negative pivots (tests/test_lu_blockdiag.py)
        from test_lu_blockdiag import edge_case_batch
        species = int(rng.integers(4, 40))
        k = int(rng.integers(1, min(12, 1024 // species) + 1))
        cells = int(rng.integers(1, 60))
        kind = (Strategy.BlockCells, Strategy.OneCell, Strategy.MultiCells)[int(rng.integers(0, 3))]
        # (not replayed: a non-finite value in a Multi-cells system too large to densify)
        nonfinite = rng.random() < 0.1 and not (kind == Strategy.MultiCells and cells * species > 2048)
        rp, ci, v, b = edge_case_batch(rng, species, cells, k, nonfinite=nonfinite,
                                       density=float(rng.uniform(0.3, 0.9)))
        return (f"edge{species}", rp, ci, v, b, kind, k if kind == Strategy.BlockCells else None,
                Algo.BICG if rng.random() < 0.5 else Algo.BICGSTAB_JACOBI, 1e-30, int(rng.integers(5, 60)))
    if rng.random() < 0.5:
        species = int(rng.choice([16, 24, 40, 64, 100, 156, 200, 312]))
        m = Mechanism(species, 3 * species, int(rng.integers(0, 5)))
        cells = int(rng.integers(1, 3000 if species <= 156 else 800))
        h = float(rng.choice([1.0, 10.0, 120.0]))
        v, b = m.newton_batch(0, cells, cells, h)
        rp, ci = m.row_ptr, m.col_idx
        src = f"M{species} h={h:g}"
    else:
        species = int(rng.integers(2, 300))
        cells = int(rng.integers(1, 400))
        rp, ci, v, b = random_batch(rng, cells, species, float(rng.uniform(0.02, 0.3)))
        src = f"rand{species}"
    kmax = max(1, 1024 // species)
    kinds = [(Strategy.BlockCells, 1), (Strategy.BlockCells, None), (Strategy.OneCell, None),
             (Strategy.BlockCells, int(rng.integers(1, kmax + 1)))]
    if cells * species <= 4000:  # a Multi-cells breakdown makes the oracle densify the whole system
        kinds.append((Strategy.MultiCells, None))
    if cells <= 2000:
        kinds.append((Strategy.ThreadPerCell, None))
    kind, k = kinds[int(rng.integers(0, len(kinds)))]
    algo = Algo.BICGSTAB_JACOBI if rng.random() < 0.6 else Algo.BICG
    tol = float(rng.choice([1e-30, 1e-12, 1e-8]))
    max_iter = int(rng.choice([5, 50, 300, 1000]))
    return src, rp, ci, v, b, kind, k, algo, tol, max_iter


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    solver = Solver(0)
    sets = {2: DeviceSet([0, 0]), 3: DeviceSet([0, 0, 0])}
    t0, n, bad = time.time(), 0, 0
    while time.time() - t0 < budget:
        src, rp, ci, v, b, kind, k, algo, tol, max_iter = case(rng)
        species, cells = len(rp) - 1, v.shape[0]
        lat = str(rng.choice(["default", "default", "1", "0"]))
        front = int(rng.choice([1, 1, 2, 3]))
        if lat == "default":
            os.environ.pop("BC_LATENCY", None)
        else:
            os.environ["BC_LATENCY"] = lat
        label = (f"{src} cells={cells} {kind.name}({k}) {algo.name} tol={tol:g} it={max_iter} latency={lat} "
                 f"devices={front}")
        st, res = of.orc_solve_batch(STRAT_ORC[kind], int(algo), 0 if k is None else k, rp, ci, v, b, tol, max_iter,
                                     workers=16)
        try:
            api = solver if front == 1 else sets[front]
            rep = api.run_strategy(BatchedSystem(species, cells, rp, ci, v, b), StrategyConfig(kind, k),
                                   DeviceSpec(), tol, max_iter, 1, algo)
            label += f" kernels={rep.kernels}"
            err = None
        except Exception as e:  # noqa: BLE001
            err = type(e).__name__
        n += 1
        if st != 0:
            ok = err is not None
            msg = f"oracle status {st}, device {err}"
        elif err is not None:
            ok, msg = False, f"device raised {err}"
        else:
            checks = {
                "x": (of.bits(np.asarray(rep.per_cell_x)) == of.bits(res.x)).all(),
                "iters": (np.asarray(rep.per_block_iterations) == res.iters).all(),
                "rms": (of.bits(np.asarray(rep.per_block_residual_rms)) == of.bits(res.rms)).all(),
                "flags": (np.asarray(rep.per_block_flags) == res.flags).all(),
                "fallbacks": rep.breakdown_fallbacks == res.report.breakdown_fallbacks,
            }
            ok = all(checks.values())
            msg = "ok" if ok else "MISMATCH " + ",".join(kk for kk, vv in checks.items() if not vv)
        bad += not ok
        print(f"{'PASS' if ok else 'FAIL'} {label}: {msg}", flush=True)
    print(f"fuzz: {n} cases, {bad} failures, {time.time() - t0:.0f} s", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
