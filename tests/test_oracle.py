"""CPU: pin the C restatement (oracle/liborc.so) against the reference --
the committed golden fixtures (always) and the live compiled reference
(oracle/_ref, when /root/reference was available to build it)."""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

import oracle_ffi as of
from fixtures import random_batch

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "m156_*.npz")) +
                                        glob.glob(os.path.join(GOLD, "random_*.npz")) +
                                        glob.glob(os.path.join(GOLD, "breakdown_*.npz"))),
                         ids=lambda p: os.path.basename(p))
def test_oracle_matches_golden(path):
    g = np.load(path)
    st, res = of.orc_solve_batch(int(g["strategy"]), 0, int(g["k"]), g["row_ptr"], g["col_idx"], g["values"],
                                 g["rhs"], float(g["tol"]), int(g["max_iter"]), workers=4)
    assert st == 0
    np.testing.assert_array_equal(of.bits(res.x), of.bits(g["x"]))
    np.testing.assert_array_equal(res.iters, g["group_iters"])
    r = res.report
    assert r.iterations_effective == int(g["iterations_effective"])
    assert r.iterations_sum == int(g["iterations_sum"])
    assert of.bits(r.max_residual_rms) == of.bits(g["max_residual_rms"])
    assert r.breakdown_fallbacks == int(g["breakdown_fallbacks"])
    assert r.cells_per_block == float(g["cells_per_block"])


def test_tree_and_plan_reduce_golden():
    g = np.load(os.path.join(GOLD, "reductions.npz"))
    off = 0
    for i, n in enumerate(g["lengths"]):
        x = g["values"][off:off + n]
        off += n
        P = 1 if n <= 1 else 1 << int(np.ceil(np.log2(n)))
        slots = np.zeros(P)
        slots[:n] = x
        got = of.orc().orc_tree_reduce_in_place(of.ptr(slots), P)
        assert of.bits(got) == of.bits(g["tree"][i]), n
        bw = int(g["plan_width"][i])
        ranges = np.array([[s, min(n, s + bw)] for s in range(0, n, bw)], np.int64)
        scratch = np.zeros(2048)
        got = of.orc().orc_plan_reduce(of.ptr(np.ascontiguousarray(x)), n, of.ptr(ranges.reshape(-1)), len(ranges),
                                       of.ptr(scratch), None)
        assert of.bits(got) == of.bits(g["plan"][i]), n


def test_lu_golden():
    g = np.load(os.path.join(GOLD, "lu.npz"))
    for i in range(4):
        st, x = of.lu_solve("orc", g[f"rp{i}"], g[f"ci{i}"], g[f"v{i}"], g[f"b{i}"])
        assert st == 0
        np.testing.assert_array_equal(of.bits(x), of.bits(g[f"x{i}"]))


def test_singular_lu_reports_error():
    rp = np.array([0, 1, 2], np.int32)
    ci = np.array([0, 0], np.int32)
    st, _ = of.lu_solve("orc", rp, ci, np.array([1.0, 2.0]), np.ones(2))
    assert st == -4  # SingularMatrix


def test_bicgstab_converges_to_lu_solution():
    """No reference BiCGSTAB exists: cross-check the restatement against the
    reference's dense LU on converging systems."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = int(rng.integers(3, 80))
        rp, ci, v, b = random_batch(rng, 1, n, 0.2)
        st, x, out = of.orc_solve_single(1, rp, ci, v[0], b[0], None, 1e-13, 10 * n)
        assert st == 0 and out.converged and not out.breakdown
        _, xl = of.lu_solve("orc", rp, ci, v[0], b[0])
        assert np.abs(x - xl).max() <= 1e-10 * max(1.0, np.abs(xl).max())


def test_bicgstab_identity_and_zero_rhs():
    n = 5
    rp = np.arange(n + 1, dtype=np.int32)
    ci = np.arange(n, dtype=np.int32)
    b = np.array([1.0, -2.0, 3.0, 0.5, 4.0])
    st, x, out = of.orc_solve_single(1, rp, ci, np.ones(n), b, None, 1e-30, 100)
    assert st == 0 and out.converged and out.iterations == 1
    np.testing.assert_array_equal(of.bits(x), of.bits(b))
    st, x, out = of.orc_solve_single(1, rp, ci, np.ones(n), np.zeros(n), None, 1e-30, 100)
    assert out.converged and out.iterations == 0


def test_argument_errors():
    rp = np.arange(3, dtype=np.int32)
    ci = np.arange(2, dtype=np.int32)
    assert of.orc_solve_single(0, rp, ci, np.ones(2), np.ones(2), None, 0.0, 10)[0] == -1
    assert of.orc_solve_single(0, rp, ci, np.ones(2), np.ones(2), None, 1e-8, 0)[0] == -1
    assert of.orc_solve_single(0, rp, ci, np.ones(2), np.ones(2), None, 1e-8, 10, [[0, 1]])[0] == -1
    v = np.ones((4, 2))
    b = np.ones((4, 2))
    assert of.orc_solve_batch(2, 0, 600, rp, ci, v, b, 1e-8, 10)[0] == -2  # InvalidGrouping
    assert of.orc_solve_batch(2, 0, 1, rp, ci, v, b, 1e-8, 10, mtpb=1)[0] == -3  # UnsupportedMechanism


def test_worker_count_never_changes_results():
    rng = np.random.default_rng(13)
    rp, ci, v, b = random_batch(rng, 9, 14)
    _, r1 = of.orc_solve_batch(2, 1, 2, rp, ci, v, b, 1e-13, 300, workers=1)
    _, r4 = of.orc_solve_batch(2, 1, 2, rp, ci, v, b, 1e-13, 300, workers=4)
    np.testing.assert_array_equal(of.bits(r1.x), of.bits(r4.x))
    np.testing.assert_array_equal(r1.iters, r4.iters)


# --- live reference (oracle/_ref) ------------------------------------------

needs_ref = pytest.mark.skipif(not of.have_ref(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_oracle_bitwise_vs_reference_random(seed):
    rng = np.random.default_rng(100 + seed)
    cells = int(rng.integers(1, 30))
    species = int(rng.integers(2, 50))
    rp, ci, v, b = random_batch(rng, cells, species, float(rng.uniform(0.05, 0.5)))
    kmax = max(1, 1024 // species)
    for strategy, k in [(0, 0), (1, 0), (2, 0), (2, 1), (2, int(rng.integers(1, min(cells, kmax) + 1)))]:
        for mtpb in (1024, 256):
            if species > mtpb:
                continue
            if strategy == 2 and k * species > mtpb:
                continue
            st1, r1 = of.ref_solve_batch(strategy, k, rp, ci, v, b, 1e-12, 400, mtpb=mtpb)
            st2, r2 = of.orc_solve_batch(strategy, 0, k, rp, ci, v, b, 1e-12, 400, mtpb=mtpb)
            assert st1 == st2 == 0
            np.testing.assert_array_equal(of.bits(r1.x), of.bits(r2.x))
            np.testing.assert_array_equal(r1.iters, r2.iters)
            assert of.bits(r1.report.max_residual_rms) == of.bits(r2.report.max_residual_rms)
            assert r1.report.breakdown_fallbacks == r2.report.breakdown_fallbacks


@needs_ref
def test_oracle_single_system_multi_block_plan_vs_reference():
    rng = np.random.default_rng(7)
    for n in (5, 32, 100, 300):
        rp, ci, v, b = random_batch(rng, 1, n, min(0.3, 6.0 / n))
        x0 = rng.uniform(-1, 1, n)
        bw = max(1, n // 3)
        ranges = [[s, min(n, s + bw)] for s in range(0, n, bw)]
        st1, x1, o1 = of.ref_bicg_single(rp, ci, v[0], b[0], x0, 1e-13, 200, ranges, True)
        st2, x2, o2 = of.orc_solve_single(0, rp, ci, v[0], b[0], x0, 1e-13, 200, ranges)
        assert st1 == st2 == 0
        np.testing.assert_array_equal(of.bits(x1), of.bits(x2))
        assert o1.iterations == o2.iterations and o1.converged == o2.converged
        assert of.bits(o1.final_residual_rms) == of.bits(o2.final_residual_rms)


@needs_ref
def test_oracle_lu_vs_reference():
    rng = np.random.default_rng(8)
    for n in (1, 2, 9, 40, 156):
        rp, ci, v, b = random_batch(rng, 1, n, 0.4)
        st1, x1 = of.lu_solve("ref", rp, ci, v[0], b[0])
        st2, x2 = of.lu_solve("orc", rp, ci, v[0], b[0])
        assert st1 == st2 == 0
        np.testing.assert_array_equal(of.bits(x1), of.bits(x2))


# --- BiCGSTAB: the restatement against the reference's own primitives ------


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_bicgstab_restatement_bitwise_vs_reference_primitives(seed):
    """orc_bicgstab_solve (bc_oracle.c) == the Jacobi-BiCGSTAB composed of the
    reference's spmv / axpby / plan_reduce_map / lu_solve and its strategy
    drivers (oracle/ref_bicgstab.cpp), for every strategy and plan."""
    rng = np.random.default_rng(300 + seed)
    cells = int(rng.integers(1, 30))
    species = int(rng.integers(2, 50))
    rp, ci, v, b = random_batch(rng, cells, species, float(rng.uniform(0.05, 0.5)))
    kmax = max(1, 1024 // species)
    for strategy, k in [(0, 0), (1, 0), (2, 0), (2, 1), (2, int(rng.integers(1, min(cells, kmax) + 1)))]:
        for mtpb in (1024, 256):
            if species > mtpb or (strategy == 2 and k * species > mtpb):
                continue
            for tol, mi in ((1e-12, 400), (1e-30, 60)):
                st1, r1 = of.ref_solve_batch_bicgstab(strategy, k, rp, ci, v, b, tol, mi, mtpb=mtpb, workers=3)
                st2, r2 = of.orc_solve_batch(strategy, 1, k, rp, ci, v, b, tol, mi, mtpb=mtpb)
                assert st1 == st2 == 0
                np.testing.assert_array_equal(of.bits(r1.x), of.bits(r2.x))
                np.testing.assert_array_equal(r1.iters, r2.iters)
                np.testing.assert_array_equal(of.bits(r1.rms), of.bits(r2.rms))
                np.testing.assert_array_equal(r1.flags, r2.flags)
                assert r1.report.breakdown_fallbacks == r2.report.breakdown_fallbacks
                assert r1.report.iterations_sum == r2.report.iterations_sum


@needs_ref
def test_bicgstab_single_multi_block_plan_vs_reference_primitives():
    rng = np.random.default_rng(17)
    for n in (1, 5, 32, 100, 300):
        rp, ci, v, b = random_batch(rng, 1, n, min(0.3, 6.0 / n))
        x0 = rng.uniform(-1, 1, n)
        bw = max(1, n // 3)
        ranges = [[s, min(n, s + bw)] for s in range(0, n, bw)]
        for tol in (1e-13, 1e-30):
            st1, x1, o1 = of.ref_bicgstab_single(rp, ci, v[0], b[0], x0, tol, 200, ranges, True)
            st2, x2, o2 = of.orc_solve_single(1, rp, ci, v[0], b[0], x0, tol, 200, ranges)
            assert st1 == st2 == 0
            np.testing.assert_array_equal(of.bits(x1), of.bits(x2))
            assert (o1.iterations, o1.converged, o1.breakdown) == (o2.iterations, o2.converged, o2.breakdown)
            assert of.bits(o1.final_residual_rms) == of.bits(o2.final_residual_rms)


@needs_ref
@pytest.mark.parametrize("h,tol", [(120.0, 1e-30), (1.0, 1e-10)])
def test_bicgstab_restatement_vs_reference_primitives_m156(m156, h, tol):
    """CB05-sized M156 cells in both regimes (P: 1000 iterations, breakdowns
    included; C: converging), Block-cells(1) and Block-cells(N)."""
    v, b = m156.newton_batch(0, 24, 100_000, h)
    for k in (1, 0):
        st1, r1 = of.ref_solve_batch_bicgstab(2, k, m156.row_ptr, m156.col_idx, v, b, tol, 1000, workers=8)
        st2, r2 = of.orc_solve_batch(2, 1, k, m156.row_ptr, m156.col_idx, v, b, tol, 1000, workers=8)
        assert st1 == st2 == 0
        np.testing.assert_array_equal(of.bits(r1.x), of.bits(r2.x))
        np.testing.assert_array_equal(r1.iters, r2.iters)
        np.testing.assert_array_equal(of.bits(r1.rms), of.bits(r2.rms))
        np.testing.assert_array_equal(r1.flags, r2.flags)


@needs_ref
def test_bicgstab_north_star_tolerance_vs_reference_lu(m156):
    """North star: converged Jacobi-BiCGSTAB solutions within 1e-10 relative
    of the reference's dense LU (dense_lu.cpp:18-63) on C-regime M156 cells."""
    v, b = m156.newton_batch(0, 40, 40, 1.0)
    st, r = of.ref_solve_batch_bicgstab(2, 1, m156.row_ptr, m156.col_idx, v, b, 1e-10, 1000, workers=8)
    assert st == 0
    ok = 0
    for c in range(40):
        if not (r.flags[c] & 1):
            continue
        st, xl = of.lu_solve("ref", m156.row_ptr, m156.col_idx, v[c], b[c])
        assert st == 0
        rel = np.abs(r.x[c] - xl).max() / np.abs(xl).max()
        assert rel <= 1e-10, (c, rel)
        ok += 1
    assert ok >= 30


@needs_ref
def test_resident_reference_batch_matches_one_shot():
    """bench.py's reference arm: the resident BatchedSystem gives the same
    bits as the one-shot wrappers (stock BiCG run_strategy, composed BiCGSTAB)."""
    rng = np.random.default_rng(21)
    rp, ci, v, b = random_batch(rng, 23, 31, 0.2)
    rb = of.RefBatch(rp, ci, v, b)
    for k in (1, 0, 5):
        st1, r1 = rb.run(0, 2, k, 1e-12, 300, workers=4)
        st2, r2 = of.ref_solve_batch(2, k, rp, ci, v, b, 1e-12, 300, workers=2)
        assert st1 == st2 == 0
        np.testing.assert_array_equal(of.bits(r1.x), of.bits(r2.x))
        np.testing.assert_array_equal(r1.iters, r2.iters)
        st1, r1 = rb.run(1, 2, k, 1e-12, 300, workers=4)
        st2, r2 = of.ref_solve_batch_bicgstab(2, k, rp, ci, v, b, 1e-12, 300, workers=1)
        assert st1 == st2 == 0
        np.testing.assert_array_equal(of.bits(r1.x), of.bits(r2.x))
        np.testing.assert_array_equal(r1.flags, r2.flags)
        np.testing.assert_array_equal(of.bits(r1.rms), of.bits(r2.rms))
    rb.close()
