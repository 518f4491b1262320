"""Small solves through every device kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/sanitize.sh).  Each case is checked
bit for bit against the oracle, so a sanitizer run is also a parity run.
    python tools/sanitize_cases.py [case ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_ffi as of  # noqa: E402
from paper_2405_17363_b200 import (Algo, BatchedSystem, DeviceSpec, Mechanism, Solver, Strategy,  # noqa: E402
                                   StrategyConfig)

S = {"one": Strategy.OneCell, "multi": Strategy.MultiCells, "block": Strategy.BlockCells,
     "thread": Strategy.ThreadPerCell}
# name: (env, strategy, k, algo, cells, h, tol, max_iter)
CASES = {
    "tmem_bicgstab": ({"BC_LATENCY": "0"}, "block", 1, 1, 40, 1.0, 1e-10, 60),
    "tmem_bicg": ({"BC_LATENCY": "0"}, "block", 1, 0, 40, 1.0, 1e-10, 60),
    "tmem_team2": ({"BC_LATENCY": "0", "BC_TMEM_TEAM": "2"}, "block", 1, 1, 20, 1.0, 1e-10, 40),
    "tmem_team4_coupled": ({"BC_LATENCY": "0"}, "block", 0, 1, 12, 1.0, 1e-10, 40),
    "latency_bicgstab": ({"BC_LATENCY": "1"}, "block", 1, 1, 10, 1.0, 1e-10, 60),
    "latency_bicg": ({"BC_LATENCY": "1"}, "block", 1, 0, 10, 1.0, 1e-10, 60),
    "v1_bicg": ({"BC_KERNEL": "v1", "BC_LATENCY": "0"}, "block", 1, 0, 20, 1.0, 1e-10, 40),
    "v1_bicgstab": ({"BC_KERNEL": "v1", "BC_LATENCY": "0"}, "block", 1, 1, 20, 1.0, 1e-10, 40),
    "multi_cells": ({}, "multi", 0, 0, 8, 1.0, 1e-10, 40),
    "thread_per_cell": ({}, "thread", 0, 1, 64, 1.0, 1e-10, 60),
    "lu_blockdiag": ({"BC_LATENCY": "0"}, "block", 0, 1, 12, 120.0, 1e-30, 1000),
    "lu_dense": ({"BC_LATENCY": "0"}, "block", 1, 1, 3, 120.0, 1e-30, 1000),
}


def run(name):
    env, strat, k, algo, cells, h, tol, mi = CASES[name]
    for key in ("BC_LATENCY", "BC_KERNEL", "BC_TMEM_TEAM"):
        os.environ.pop(key, None)
    os.environ.update(env)
    m = Mechanism(156, 468, 0)
    first = 213 if name == "lu_dense" else 0  # cell 214 of 100k breaks down in the P regime (dense LU path)
    v, b = m.newton_batch(first, cells, 100_000, h)
    s = Solver(0)
    rep = s.run_strategy(BatchedSystem(156, cells, m.row_ptr, m.col_idx, v, b), StrategyConfig(S[strat], k or None),
                         DeviceSpec(), tol, mi, 1, Algo(algo))
    st, res = of.orc_solve_batch({"one": 0, "multi": 1, "block": 2, "thread": 0}[strat], algo, k, m.row_ptr,
                                 m.col_idx, v, b, tol, mi, workers=4)
    ok = st == 0 and np.array_equal(of.bits(np.asarray(rep.per_cell_x)), of.bits(res.x)) and \
        np.array_equal(np.asarray(rep.per_block_iterations), res.iters)
    print(f"{name}: kernels={rep.kernels} fallbacks={rep.breakdown_fallbacks} bitwise={'yes' if ok else 'NO'}",
          flush=True)
    if not ok and st == 0:
        xg = np.asarray(rep.per_cell_x)
        bad = (of.bits(xg) != of.bits(res.x))
        print(f"  x mismatches {int(bad.sum())} of {bad.size}; iterations gpu {list(rep.per_block_iterations)[:4]} "
              f"oracle {list(res.iters)[:4]}; max rel {float(np.abs(xg - res.x).max() / np.abs(res.x).max()):.3e}",
              flush=True)
    s.close()
    return ok


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    sys.exit(0 if all([run(n) for n in names]) else 1)
