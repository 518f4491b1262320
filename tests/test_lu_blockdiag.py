"""Breakdown fallback of coupled Block-cells(k) groups (strategies.cpp:46-60).
The reference densifies a k-cell group and runs dense_lu.cpp's O((k s)^3) LU
on the block-diagonal matrix; the device factors the k diagonal blocks one by
one and replays the only effect the zero off-diagonal blocks have -- the sign
of zeros (csrc/bc_lu.cuh).  These cases are built to exercise exactly that:
every group breaks down at BiCG's first iteration (b = e_i on rows whose
diagonal is a signed zero, so <p~, A p> = a_ii = 0 exactly), the other cells
have all-zero right-hand sides of mixed sign (their solutions are signed
zeros), matrices carry -0.0 entries and negative pivots, plus a few
non-finite groups that must take the dense path.  Bitwise against the
compiled reference (oracle/_ref) and the C restatement."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_ffi as of
from paper_2405_17363_b200 import Algo, BatchedSystem, DeviceSpec, Strategy, StrategyConfig


def edge_case_batch(rng, species, cells, k, nonfinite=False, density=0.45):
    n = species
    dense = rng.random((n, n)) < density
    np.fill_diagonal(dense, True)
    rows, cols = np.nonzero(dense)
    row_ptr = np.zeros(n + 1, np.int32)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    col_idx = cols.astype(np.int32)
    nnz = len(col_idx)
    diag_pos = np.array([row_ptr[i] + np.nonzero(col_idx[row_ptr[i]:row_ptr[i + 1]] == i)[0][0] for i in range(n)])
    v = rng.uniform(-1.0, 1.0, (cells, nnz))
    v[rng.random((cells, nnz)) < 0.15] = -0.0
    v[rng.random((cells, nnz)) < 0.05] = 0.0
    # diagonals of either sign (negative pivots), large enough to stay regular
    v[:, diag_pos] = rng.uniform(1.0, 3.0, (cells, n)) * rng.choice([-1.0, 1.0], (cells, n)) * 0.5 * n
    b = np.where(rng.random((cells, n)) < 0.5, -0.0, 0.0)
    zero_row = int(rng.integers(0, n))
    for g0 in range(0, cells, k):
        active = [c for c in range(g0, min(cells, g0 + k)) if rng.random() < 0.5] or [g0]
        for c in active:
            v[c, diag_pos[zero_row]] = -0.0 if rng.random() < 0.5 else 0.0
            b[c, zero_row] = rng.uniform(0.5, 2.0) * rng.choice([-1.0, 1.0])
    if nonfinite:
        v[int(rng.integers(0, cells)), int(rng.integers(0, nnz))] = np.inf
    return row_ptr, col_idx, v, b


def ref_or_oracle(rp, ci, v, b, k, algo):
    if algo == Algo.BICG and of.have_ref():
        st, res = of.ref_solve_batch(2, k, rp, ci, v, b, 1e-30, 40)  # one worker: the reference terminates on a worker-thread throw
        return st, res
    return of.orc_solve_batch(2, int(algo), k, rp, ci, v, b, 1e-30, 40)


def edge_case(seed):
    rng = np.random.default_rng(1000 + seed)
    species = int(rng.choice([6, 8, 11, 16]))
    k = int(rng.integers(2, 7))
    cells = k * int(rng.integers(2, 6)) + int(rng.integers(0, k))
    return (species, k, cells) + edge_case_batch(rng, species, cells, k, nonfinite=seed % 6 == 5)


def test_oracle_edge_cases_match_reference():
    """CPU: the restatement's dense LU fallback equals the reference's on every
    case below (breakdowns, signed-zero solutions, singular groups, NaN)."""
    if not of.have_ref():
        pytest.skip("oracle/_ref not built")
    for seed in range(24):
        species, k, cells, rp, ci, v, b = edge_case(seed)
        st_r, want = of.ref_solve_batch(2, k, rp, ci, v, b, 1e-30, 40)
        st_o, got = of.orc_solve_batch(2, int(Algo.BICG), k, rp, ci, v, b, 1e-30, 40)
        assert st_r == st_o
        if st_r == 0:
            assert want.report.breakdown_fallbacks > 0
            np.testing.assert_array_equal(of.bits(got.x), of.bits(want.x))
            np.testing.assert_array_equal(got.iters, want.iters)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(24))
def test_coupled_group_lu_signed_zeros_bitwise(solver, seed):
    species, k, cells, rp, ci, v, b = edge_case(seed)
    for algo in (Algo.BICG, Algo.BICGSTAB_JACOBI):
        st, want = ref_or_oracle(rp, ci, v, b, k, algo)
        sysm = BatchedSystem(species, cells, rp, ci, v, b)
        try:
            rep = solver.run_strategy(sysm, StrategyConfig(Strategy.BlockCells, k), DeviceSpec(), 1e-30, 40, 1, algo)
            err = None
        except Exception as e:  # noqa: BLE001
            err = type(e).__name__
        if st == -4:
            assert err == "SingularMatrix", (seed, algo, err)
            continue
        assert st == 0 and err is None, (seed, algo, st, err)
        np.testing.assert_array_equal(of.bits(rep.per_cell_x), of.bits(want.x), err_msg=f"seed {seed} {algo}")
        np.testing.assert_array_equal(np.asarray(rep.per_block_iterations), want.iters)
        if algo == Algo.BICG:
            assert rep.breakdown_fallbacks == want.report.breakdown_fallbacks > 0


@pytest.mark.gpu
def test_block_cells_n_breakdown_groups_m156(solver):
    """Coupled 936-row M156 groups in the P regime (most break down under
    Jacobi-BiCGSTAB): the block-diagonal LU against the oracle's dense LU."""
    from paper_2405_17363_b200 import Mechanism
    m = Mechanism(156, 468, 0)
    v, bb = m.newton_batch(0, 48, 48, 120.0)
    sysm = BatchedSystem(156, 48, m.row_ptr, m.col_idx, v, bb)
    rep = solver.run_strategy(sysm, StrategyConfig(Strategy.BlockCells, 6), DeviceSpec(), 1e-30, 1000, 1,
                              Algo.BICGSTAB_JACOBI)
    st, want = of.orc_solve_batch(2, int(Algo.BICGSTAB_JACOBI), 6, m.row_ptr, m.col_idx, v, bb, 1e-30, 1000,
                                  workers=8)
    assert st == 0 and want.report.breakdown_fallbacks > 0
    np.testing.assert_array_equal(of.bits(rep.per_cell_x), of.bits(want.x))
    np.testing.assert_array_equal(of.bits(rep.per_block_residual_rms), of.bits(want.rms))
    np.testing.assert_array_equal(rep.per_block_flags, want.flags)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(2))
def test_multi_cells_large_breakdown_sign_chain(solver, seed):
    """Multi-cells over 300 cells (2,400 rows): one system too large to densify,
    so the device solves it cell by cell and the host replays the cross-cell
    sign-of-zero chain (bc_capi.cu lu_sign_chain).  Bitwise against the
    oracle's dense 2400^2 LU (dense_lu.cpp), which differs from independent
    per-cell LUs in the sign of zeros on these inputs."""
    rng = np.random.default_rng(seed)
    rp, ci, v, b = edge_case_batch(rng, 8, 300, 300, density=0.9)
    st, want = of.orc_solve_batch(1, int(Algo.BICG), 0, rp, ci, v, b, 1e-30, 40, workers=8)
    assert st == 0 and want.report.breakdown_fallbacks == 1
    per_cell = np.stack([of.lu_solve("orc", rp, ci, v[c], b[c])[1] for c in range(300)])
    assert (of.bits(per_cell) != of.bits(want.x)).any()  # the chain matters here
    sysm = BatchedSystem(8, 300, rp, ci, v, b)
    rep = solver.run_strategy(sysm, StrategyConfig(Strategy.MultiCells), DeviceSpec(), 1e-30, 40, 1, Algo.BICG)
    np.testing.assert_array_equal(of.bits(rep.per_cell_x), of.bits(want.x))
    assert of.bits(rep.max_residual_rms) == of.bits(want.report.max_residual_rms)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [None])  # k = 3 coupled 312-row blocks: these 9 cells break down
def test_coupled_breakdown_blocks_above_256_rows(solver, k):
    """Coupled groups of 312-species cells (blocks above 256 rows: the back
    substitution's long-row path) breaking down in the P regime -- the cases
    the round-2 fuzzer caught (tools/fuzz_gpu.py seed 41)."""
    from paper_2405_17363_b200 import Mechanism, REGIME_P
    m = Mechanism(312, 936, 0)
    v, b = m.newton_batch(0, 9, 100_000, REGIME_P.h)
    rep = solver.run_strategy(BatchedSystem(312, 9, m.row_ptr, m.col_idx, v, b), StrategyConfig(Strategy.BlockCells, k),
                              DeviceSpec(), 1e-30, 300, 1, Algo.BICGSTAB_JACOBI)
    assert rep.breakdown_fallbacks >= 1
    st, res = of.orc_solve_batch(2, 1, 0 if k is None else k, m.row_ptr, m.col_idx, v, b, 1e-30, 300, workers=8)
    assert st == 0
    np.testing.assert_array_equal(of.bits(np.asarray(rep.per_cell_x)), of.bits(res.x))
    np.testing.assert_array_equal(of.bits(np.asarray(rep.per_block_residual_rms)), of.bits(res.rms))
    np.testing.assert_array_equal(np.asarray(rep.per_block_iterations), res.iters)
