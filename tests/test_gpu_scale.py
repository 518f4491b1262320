"""Parity at the configurations that carry the metric (BASELINE.json configs
1-4), against the strongest checker: Jacobi-BiCGSTAB composed from the
reference's own primitives (oracle/_ref), BiCG through the reference's
run_strategy, the C restatement only where oracle/_ref is absent.  Exercises
the paths that exist only at scale: many TMEM waves and the atomic group
counter, the streamed host-input gate (32 chunks), the LU fallback batch, and
a 1M-cell launch (checked on a strided sample of whole groups)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_ffi as of
from paper_2405_17363_b200 import (KERNEL_TMEM, Algo, BatchedSystem, DeviceSpec, Mechanism, REGIME_P, Strategy,
                                   StrategyConfig)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def check(rep, idx, v, b, row_ptr, col_idx, algo, k, reg, label):
    """Compare cells `idx` (whole groups, in order) of a GPU report with the checker."""
    if of.have_ref():
        rb = of.RefBatch(row_ptr, col_idx, np.ascontiguousarray(v[idx]), np.ascontiguousarray(b[idx]))
        st, res = rb.run(int(algo), 2, k, reg.tol, reg.max_iter, workers=0)
        rb.close()
    else:
        st, res = of.orc_solve_batch(2, int(algo), k, row_ptr, col_idx, np.ascontiguousarray(v[idx]),
                                     np.ascontiguousarray(b[idx]), reg.tol, reg.max_iter, workers=16)
    assert st == 0
    x = rep.per_cell_x.cpu().numpy() if hasattr(rep.per_cell_x, "cpu") else np.asarray(rep.per_cell_x)
    np.testing.assert_array_equal(of.bits(x[idx]), of.bits(res.x), err_msg=f"{label}: x bits")
    g = idx[::k] // k
    np.testing.assert_array_equal(np.asarray(rep.per_block_iterations)[g], res.iters, err_msg=f"{label}: iterations")
    if res.rms is not None:
        np.testing.assert_array_equal(of.bits(np.asarray(rep.per_block_residual_rms)[g]), of.bits(res.rms),
                                      err_msg=f"{label}: rms")
        np.testing.assert_array_equal(np.asarray(rep.per_block_flags)[g], res.flags, err_msg=f"{label}: flags")


@pytest.mark.parametrize("algo", [Algo.BICGSTAB_JACOBI, Algo.BICG])
def test_10k_m156_all_cells(solver, m156, algo):
    """configs[1]: 10k cells, every cell checked; BiCGSTAB with host inputs
    (the streamed 32-chunk gate), BiCG with device inputs."""
    import torch
    cells = 10_000
    v, b = m156.newton_batch(0, cells, cells, REGIME_P.h)
    if algo == Algo.BICG:
        sysm = BatchedSystem(156, cells, m156.row_ptr, m156.col_idx, torch.from_numpy(v).cuda(),
                             torch.from_numpy(b).cuda())
    else:
        sysm = BatchedSystem(156, cells, m156.row_ptr, m156.col_idx, v, b)
    rep = solver.run_strategy(sysm, StrategyConfig(Strategy.BlockCells, 1), DeviceSpec(), REGIME_P.tol,
                              REGIME_P.max_iter, 1, algo)
    assert rep.kernels & KERNEL_TMEM
    check(rep, np.arange(cells), v, b, m156.row_ptr, m156.col_idx, algo, 1, REGIME_P, f"10k {algo.name}")


def test_m312_20k_cells(solver):
    """configs[4]: the scaled mechanism (312 species, 3032 nnz), 20k cells."""
    m = Mechanism(312, 936, 0)
    cells = 20_000
    v, b = m.newton_batch(0, cells, 100_000, REGIME_P.h)
    rep = solver.run_strategy(BatchedSystem(312, cells, m.row_ptr, m.col_idx, v, b),
                              StrategyConfig(Strategy.BlockCells, 1), DeviceSpec(), REGIME_P.tol, REGIME_P.max_iter,
                              1, Algo.BICGSTAB_JACOBI)
    check(rep, np.arange(cells), v, b, m.row_ptr, m.col_idx, Algo.BICGSTAB_JACOBI, 1, REGIME_P, "M312 20k")


def test_block_cells_n_100k_sampled(solver, m156):
    """Block-cells(N) (k = 6, 936-row coupled groups) at 100k cells: nearly
    every group falls back to the device LU; every 500th group checked (the
    checker densifies each 936-row group for its LU: ~1 GFLOP apiece)."""
    import torch
    cells, k = 100_000, 6
    v, b = m156.newton_batch(0, cells, cells, REGIME_P.h)
    rep = solver.run_strategy(BatchedSystem(156, cells, m156.row_ptr, m156.col_idx, torch.from_numpy(v).cuda(),
                                            torch.from_numpy(b).cuda()),
                              StrategyConfig(Strategy.BlockCells, None), DeviceSpec(), REGIME_P.tol, REGIME_P.max_iter,
                              1, Algo.BICGSTAB_JACOBI)
    assert rep.breakdown_fallbacks > 10_000
    groups = np.arange(0, cells // k, 500)
    idx = (groups[:, None] * k + np.arange(k)[None, :]).reshape(-1)
    check(rep, idx, v, b, m156.row_ptr, m156.col_idx, Algo.BICGSTAB_JACOBI, k, REGIME_P, "Block-cells(N) 100k")


def test_1m_cells_sampled(solver, m156):
    """configs[3]: one 1M-cell launch (an 8-GPU shard is 125k), host inputs;
    a strided 20k-cell sample checked, plus the report's totals."""
    cells = 1_000_000
    v, b = m156.newton_batch(0, cells, cells, REGIME_P.h)
    rep = solver.run_strategy(BatchedSystem(156, cells, m156.row_ptr, m156.col_idx, v, b),
                              StrategyConfig(Strategy.BlockCells, 1), DeviceSpec(), REGIME_P.tol, REGIME_P.max_iter,
                              1, Algo.BICGSTAB_JACOBI)
    assert len(rep.per_block_iterations) == cells
    assert rep.iterations_sum == int(np.asarray(rep.per_block_iterations).sum())
    idx = np.arange(7, cells, 50)
    check(rep, idx, v, b, m156.row_ptr, m156.col_idx, Algo.BICGSTAB_JACOBI, 1, REGIME_P, "1M sampled")
