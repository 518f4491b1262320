"""Randomised shapes through every TMEM-kernel path (one warp, two- and
four-warp teams, BiCG pair schedules, coupled Block-cells(k) groups, batch
sizes that pick different team widths), bit for bit against the C oracle.
Mechanisms of 24..300 species with the synthetic generator's sparsity, and
random diagonally dominant patterns."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_ffi as of
from fixtures import random_batch
from paper_2405_17363_b200 import KERNEL_LATENCY, KERNEL_TMEM, Algo, BatchedSystem, DeviceSpec, Mechanism, Strategy, StrategyConfig

pytestmark = pytest.mark.gpu


def check(solver, rp, ci, v, b, k, algo, tol, max_iter):
    sysm = BatchedSystem(len(rp) - 1, v.shape[0], rp, ci, v, b)
    rep = solver.run_strategy(sysm, StrategyConfig(Strategy.BlockCells, k), DeviceSpec(), tol, max_iter, 1, algo)
    st, res = of.orc_solve_batch(2, int(algo), 0 if k is None else k, rp, ci, v, b, tol, max_iter, workers=8)
    assert st == 0
    np.testing.assert_array_equal(of.bits(rep.per_cell_x), of.bits(res.x))
    np.testing.assert_array_equal(np.asarray(rep.per_block_iterations), res.iters)
    np.testing.assert_array_equal(of.bits(rep.per_block_residual_rms), of.bits(res.rms))
    np.testing.assert_array_equal(rep.per_block_flags, res.flags)
    return rep


@pytest.mark.parametrize("species,seed", [(24, 11), (70, 12), (130, 13), (200, 14), (300, 15)])
def test_generated_mechanisms_every_grouping(solver, species, seed):
    m = Mechanism(species, 3 * species, seed)
    rng = np.random.default_rng(seed)
    for cells, k in ((37, 1), (700, 1), (2000, 1), (23, None), (41, 2)):
        if k is not None and k * species > 1024:
            continue
        v, b = m.newton_batch(0, cells, cells, 1.0)
        for algo in (Algo.BICGSTAB_JACOBI, Algo.BICG):
            rep = check(solver, m.row_ptr, m.col_idx, v, b, k, algo, 1e-10, int(rng.integers(40, 400)))
            n = species * (k if k else 1024 // species)
            if k == 1 and n >= 65:  # one-cell groups with an instance: TMEM, or latency mode for small batches
                assert rep.kernels & (KERNEL_TMEM | KERNEL_LATENCY), (species, cells, k, algo, rep.kernels)


@pytest.mark.parametrize("seed", range(4))
def test_random_patterns_large(solver, seed):
    rng = np.random.default_rng(100 + seed)
    species = int(rng.integers(65, 260))
    cells = int(rng.integers(5, 60))
    rp, ci, v, b = random_batch(rng, cells, species, float(rng.uniform(0.01, 0.08)))
    for k in (1, int(rng.integers(2, max(3, 1024 // species + 1))), None):
        if k is not None and k * species > 1024:
            continue
        for algo in (Algo.BICGSTAB_JACOBI, Algo.BICG):
            check(solver, rp, ci, v, b, k, algo, 1e-12, 120)


@pytest.mark.parametrize("species,k", [(1024, 1), (512, 2), (128, 8), (341, 3), (33, 31)])
def test_largest_groups(solver, species, k):
    """Groups of exactly (or just under) the 1024-row limit (exec_model.cpp:
    k * s <= 1024): the four-warp TMEM teams' widest trees, both algorithms."""
    rng = np.random.default_rng(species * 7 + k)
    rp, ci, v, b = random_batch(rng, 2 * k + 1, species, 4.0 / species)
    for algo in (Algo.BICGSTAB_JACOBI, Algo.BICG):
        rep = check(solver, rp, ci, v, b, k, algo, 1e-12, 60)
        assert len(rep.per_block_iterations) == 3
