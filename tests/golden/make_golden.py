"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libbcref.so, built by oracle/Makefile from /root/reference).

Run from the repo root:  python tests/golden/make_golden.py
The fixtures pin the oracle (and through it the CUDA path) on machines where
/root/reference is absent (the GPU box).  Each .npz holds the inputs and the
reference's outputs; float arrays are compared bitwise by the tests.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_ffi as of  # noqa: E402
from fixtures import random_batch  # noqa: E402
from paper_2405_17363_b200.workload import Mechanism  # noqa: E402


def strategy_case(name, strategy, k, rp, ci, v, b, tol, max_iter):
    st, res = of.ref_solve_batch(strategy, k, rp, ci, v, b, tol, max_iter, workers=4)
    assert st == 0, (name, st)
    r = res.report
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), row_ptr=rp, col_idx=ci, values=v, rhs=b,
                        strategy=strategy, k=k, tol=tol, max_iter=max_iter, x=res.x, group_iters=res.iters,
                        iterations_effective=r.iterations_effective, iterations_sum=r.iterations_sum,
                        max_residual_rms=r.max_residual_rms, breakdown_fallbacks=r.breakdown_fallbacks,
                        cells_per_block=r.cells_per_block)
    print(f"{name}: groups={r.n_groups} it_eff={r.iterations_effective} fb={r.breakdown_fallbacks}")


def main():
    assert of.have_ref(), "build oracle/_ref first: make -C oracle"
    m = Mechanism(156, 468, 0)
    # M156 first Newton systems: C regime (converging) and P regime (capped)
    v, b = m.newton_batch(0, 8, 100, 1.0)
    for strategy, k, tag in [(2, 1, "bc1"), (2, 0, "bcN"), (1, 0, "multi"), (0, 0, "one")]:
        strategy_case(f"m156_C_{tag}", strategy, k, m.row_ptr, m.col_idx, v, b, 1e-10, 1000)
    v, b = m.newton_batch(0, 4, 100, 120.0)
    strategy_case("m156_P_bc1_it50", 2, 1, m.row_ptr, m.col_idx, v, b, 1e-30, 50)

    rng = np.random.default_rng(99)
    for i, (cells, species, k) in enumerate([(5, 11, 1), (11, 10, 10), (9, 14, 2), (90, 13, 0), (4, 20, 4)]):
        rp, ci, v, b = random_batch(rng, cells, species)
        strategy_case(f"random_{i}", 2 if k else 1, k, rp, ci, v, b, 1e-12, 500)
    # breakdown -> LU fallback (test_strategies.cpp:288-314)
    rp = np.array([0, 2, 4], np.int32)
    ci = np.array([0, 1, 0, 1], np.int32)
    v = np.array([[3.0, 1.0, -1.0, 3.0], [0.0, 1.0, -1.0, 0.0]])
    b = np.array([[1.0, 2.0], [3.0, 4.0]])
    strategy_case("breakdown_2x2", 2, 1, rp, ci, v, b, 1e-13, 100)

    # tree reduction (reduction.cpp:38-58) and plan reduce with a host stage
    vals, trees, plans = [], [], []
    for n in list(range(1, 70)) + [100, 156, 255, 256, 257, 1000, 1024, 1500]:
        x = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-5, 5, n)
        x[rng.random(n) < 0.1] = -0.0
        vals.append(x)
        trees.append(of.ref().ref_tree_reduce(of.ptr(x), n, int(2 ** np.ceil(np.log2(max(n, 1))))))
        bw = int(rng.integers(1, max(2, n)))
        ranges = np.array([[s, min(n, s + bw)] for s in range(0, n, bw)], np.int64)
        plans.append((bw, of.ref().ref_plan_reduce(of.ptr(x), n, of.ptr(ranges.reshape(-1)), len(ranges))))
    np.savez_compressed(os.path.join(HERE, "reductions.npz"), lengths=np.array([len(x) for x in vals]),
                        values=np.concatenate(vals), tree=np.array(trees),
                        plan_width=np.array([p[0] for p in plans]), plan=np.array([p[1] for p in plans]))

    # dense LU (dense_lu.cpp:18-67)
    lus = {}
    for i, n in enumerate((2, 7, 20, 64)):
        rp, ci, v, b = random_batch(rng, 1, n, 0.5)
        st, x = of.lu_solve("ref", rp, ci, v[0], b[0])
        assert st == 0
        lus.update({f"rp{i}": rp, f"ci{i}": ci, f"v{i}": v[0], f"b{i}": b[0], f"x{i}": x})
    np.savez_compressed(os.path.join(HERE, "lu.npz"), **lus)

    # workload generator (mechanism.cpp / simulate.cpp) digests
    dig = {}
    for species in (156, 312):
        nnz = of._i64()
        of.ref().ref_mechanism_pattern(species, 3 * species, 0, of.C.byref(nnz), None, None)
        rp = np.zeros(species + 1, np.int32)
        ci = np.zeros(nnz.value, np.int32)
        of.ref().ref_mechanism_pattern(species, 3 * species, 0, of.C.byref(nnz), of.ptr(rp), of.ptr(ci))
        for h in (120.0, 1.0):
            vv = np.zeros(10 * nnz.value)
            bb = np.zeros(10 * species)
            of.ref().ref_newton_batch(species, 3 * species, 0, 37, 10, 1000, 1, h, of.ptr(vv), of.ptr(bb))
            dig[f"m{species}_h{int(h)}"] = hashlib.sha256(vv.tobytes() + bb.tobytes()).hexdigest()
        dig[f"m{species}_pattern"] = hashlib.sha256(rp.tobytes() + ci.tobytes()).hexdigest()
    with open(os.path.join(HERE, "workload_digests.txt"), "w") as f:
        for k_, d in sorted(dig.items()):
            f.write(f"{k_} {d}\n")
    print("ok")


if __name__ == "__main__":
    main()
