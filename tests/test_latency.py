"""Latency mode (bc_latency.cuh): one CTA per group, one thread per row, for
batches too small to fill the GPU.  Bitwise against the oracle / the
reference for both algorithms, every group geometry it takes (P = 64..512),
and it is the kernel that runs for small batches by default."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle_ffi as of
from fixtures import random_batch
from paper_2405_17363_b200 import (KERNEL_LATENCY, Algo, BatchedSystem, DeviceSpec, Mechanism, REGIME_C, REGIME_P,
                                   Strategy, StrategyConfig)
from test_gpu_parity import assert_matches_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture
def force_latency():
    old = os.environ.get("BC_LATENCY")
    os.environ["BC_LATENCY"] = "1"
    yield
    if old is None:
        del os.environ["BC_LATENCY"]
    else:
        os.environ["BC_LATENCY"] = old


@pytest.mark.parametrize("regime", ["P", "C"])
@pytest.mark.parametrize("algo", [Algo.BICGSTAB_JACOBI, Algo.BICG])
def test_latency_m156_bitwise(solver, m156, regime, algo):
    """configs[0]: 100 CB05-sized cells -- the default path for this batch."""
    reg = REGIME_P if regime == "P" else REGIME_C
    v, b = m156.newton_batch(0, 100, 100, reg.h)
    sysm = BatchedSystem(156, 100, m156.row_ptr, m156.col_idx, v, b)
    rep = solver.run_strategy(sysm, StrategyConfig(Strategy.BlockCells, 1), DeviceSpec(), reg.tol, reg.max_iter, 1,
                              algo)
    assert rep.kernels & KERNEL_LATENCY, rep.kernels
    st, res = of.orc_solve_batch(2, int(algo), 1, m156.row_ptr, m156.col_idx, v, b, reg.tol, reg.max_iter, workers=8)
    assert st == 0
    assert_matches_oracle(rep, res, f"latency {regime} {algo}")
    if of.have_ref():
        if algo == Algo.BICG:
            st, rr = of.ref_solve_batch(2, 1, m156.row_ptr, m156.col_idx, v, b, reg.tol, reg.max_iter, workers=8)
            assert st == 0
            np.testing.assert_array_equal(of.bits(np.asarray(rep.per_cell_x)), of.bits(rr.x))
            np.testing.assert_array_equal(rep.per_block_iterations, rr.iters)
        else:
            st, rr = of.ref_solve_batch_bicgstab(2, 1, m156.row_ptr, m156.col_idx, v, b, reg.tol, reg.max_iter,
                                                 workers=8)
            assert st == 0
            assert_matches_oracle(rep, rr, f"latency {regime} vs reference primitives")


@pytest.mark.parametrize("algo", [Algo.BICGSTAB_JACOBI, Algo.BICG])
def test_latency_group_geometries(solver, force_latency, algo):
    """P = 64, 128, 256: coupled groups (k = 2, 3 of small cells), the
    remainder group, and random patterns up to 32 entries per row / column;
    P = 512 (M312, M156 k = 3) is checked to fall back to the throughput
    kernels, bit for bit all the same."""
    m312 = Mechanism(312, 936, 0)
    cases = []
    v, b = m312.newton_batch(0, 9, 9, REGIME_C.h)
    cases.append(("M312", m312.row_ptr, m312.col_idx, v, b, [1]))
    m156 = Mechanism(156, 468, 0)
    v, b = m156.newton_batch(0, 7, 7, REGIME_C.h)
    cases.append(("M156 k=3 (P=512, remainder 1)", m156.row_ptr, m156.col_idx, v, b, [3, 2]))
    rng = np.random.default_rng(11)
    for species, dens in ((40, 0.3), (100, 0.12), (60, 0.45)):
        rp, ci, v, b = random_batch(rng, 5, species, dens)
        cases.append((f"random {species}", rp, ci, v, b, [1, 2]))
    ran = 0
    for label, rp, ci, v, b, ks in cases:
        sysm = BatchedSystem(len(rp) - 1, v.shape[0], rp, ci, v, b)
        for k in ks:
            for tol, mi in ((1e-10, 400), (1e-30, 120)):
                rep = solver.run_strategy(sysm, StrategyConfig(Strategy.BlockCells, k), DeviceSpec(), tol, mi, 1,
                                          algo)
                st, res = of.orc_solve_batch(2, int(algo), k, rp, ci, v, b, tol, mi, workers=8)
                assert st == 0
                assert_matches_oracle(rep, res, f"{label} k={k} tol={tol} {algo}")
                ran += bool(rep.kernels & KERNEL_LATENCY)
    assert ran >= 10, ran
