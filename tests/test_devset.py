"""The drop-in API over several GPUs (bc_devset): contiguous
group-aligned shards, one host thread per device, report merged in group
order.  On one B200 the set lists the same GPU several times (one context
and stream each, solving concurrently); every output must equal one
context's solve bit for bit, and the reference's own C++ suite must pass
through the shim with BLOCKCELLS_B200_DEVICES set."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle_ffi as of
from fixtures import random_batch
from paper_2405_17363_b200 import (Algo, BatchedSystem, DeviceSet, DeviceSpec, Mechanism, REGIME_P, Strategy,
                                   StrategyConfig)

pytestmark = pytest.mark.gpu


def same(a, b, label):
    np.testing.assert_array_equal(of.bits(np.asarray(a.per_cell_x)), of.bits(np.asarray(b.per_cell_x)),
                                  err_msg=label)
    np.testing.assert_array_equal(a.per_block_iterations, b.per_block_iterations, err_msg=label)
    np.testing.assert_array_equal(of.bits(a.per_block_residual_rms), of.bits(b.per_block_residual_rms), err_msg=label)
    np.testing.assert_array_equal(a.per_block_flags, b.per_block_flags, err_msg=label)
    for f in ("iterations_effective", "iterations_sum", "breakdown_fallbacks", "cells_per_block"):
        assert getattr(a, f) == getattr(b, f), (label, f)
    assert of.bits(a.max_residual_rms) == of.bits(b.max_residual_rms), label


@pytest.mark.parametrize("ndev", [2, 3])
def test_device_set_equals_single_context_m156(solver, m156, ndev):
    v, b = m156.newton_batch(0, 601, 601, REGIME_P.h)
    sysm = BatchedSystem(156, 601, m156.row_ptr, m156.col_idx, v, b)
    ds = DeviceSet([0] * ndev)
    try:
        for kind, k in ((Strategy.BlockCells, 1), (Strategy.BlockCells, None), (Strategy.BlockCells, 4),
                        (Strategy.OneCell, None), (Strategy.ThreadPerCell, None), (Strategy.MultiCells, None)):
            for algo in (Algo.BICGSTAB_JACOBI, Algo.BICG):
                if kind == Strategy.MultiCells and algo == Algo.BICGSTAB_JACOBI:
                    continue  # a breakdown there densifies the whole system (test_gpu_parity covers it)
                cfg = StrategyConfig(kind, k)
                one = solver.run_strategy(sysm, cfg, DeviceSpec(), REGIME_P.tol, 150, 1, algo)
                many = ds.run_strategy(sysm, cfg, DeviceSpec(), REGIME_P.tol, 150, 1, algo)
                same(one, many, f"{ndev} devices {kind} {k} {algo}")
    finally:
        ds.close()


def test_device_set_ragged_shards_and_tiny_batches(solver):
    rng = np.random.default_rng(5)
    rp, ci, v, b = random_batch(rng, 37, 45, 0.15)
    ds = DeviceSet([0, 0, 0, 0])
    try:
        for cells in (1, 2, 5, 37):  # fewer groups than devices, remainder group on the last shard
            sysm = BatchedSystem(45, cells, rp, ci, np.ascontiguousarray(v[:cells]), np.ascontiguousarray(b[:cells]))
            for k in (1, 4, None):
                cfg = StrategyConfig(Strategy.BlockCells, k)
                for algo in (Algo.BICG, Algo.BICGSTAB_JACOBI):
                    one = solver.run_strategy(sysm, cfg, DeviceSpec(), 1e-12, 300, 1, algo)
                    many = ds.run_strategy(sysm, cfg, DeviceSpec(), 1e-12, 300, 1, algo)
                    same(one, many, f"cells {cells} k {k} {algo}")
    finally:
        ds.close()


def test_device_set_rejects_device_arrays_over_several_gpus():
    import torch
    rng = np.random.default_rng(6)
    rp, ci, v, b = random_batch(rng, 8, 20)
    ds = DeviceSet([0, 0])
    try:
        sysm = BatchedSystem(20, 8, rp, ci, torch.from_numpy(v).cuda(), torch.from_numpy(b).cuda())
        with pytest.raises(ValueError):
            ds.run_strategy(sysm, StrategyConfig(Strategy.BlockCells, 1), DeviceSpec(), 1e-10, 50)
    finally:
        ds.close()


def test_reference_suite_through_device_set():
    """The reference's own C++ unit tests (tests/cpp) through the shim with
    BLOCKCELLS_B200_DEVICES=0,0: run_strategy on a two-context device set
    reproduces the reference's outcome check for check."""
    import test_reference_suite as trs
    if not (os.path.exists(trs.B200) and os.path.exists(trs.REF)):
        pytest.skip("tests/cpp binaries not built")
    ref_counts, ref_fail, _ = trs.run(trs.REF)
    old = os.environ.get("BLOCKCELLS_B200_DEVICES")
    os.environ["BLOCKCELLS_B200_DEVICES"] = "0,0"
    try:
        counts, failures, out = trs.run(trs.B200)
    finally:
        if old is None:
            del os.environ["BLOCKCELLS_B200_DEVICES"]
        else:
            os.environ["BLOCKCELLS_B200_DEVICES"] = old
    assert counts == ref_counts, out[-3000:]
    assert failures == ref_fail, out[-3000:]


# --- torch.distributed ranks, each driving the GPU solver on its shard -------

def _rank_worker(rank, world, port, cells, k, out_path):
    import torch.distributed as dist

    from paper_2405_17363_b200 import Solver
    from paper_2405_17363_b200.sharding import merge_reports, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = Mechanism(156, 468, 0)
    first, count = shard_range(cells, k, rank, world)
    v, b = m.newton_batch(first, count, cells, REGIME_P.h)  # global cell conditions
    s = Solver(0)  # every rank on GPU 0 (this box has one)
    rep = s.run_strategy(BatchedSystem(156, count, m.row_ptr, m.col_idx, v, b), StrategyConfig(Strategy.BlockCells, k),
                         DeviceSpec(), REGIME_P.tol, 200, 1, Algo.BICGSTAB_JACOBI)
    merged = merge_reports(dict(iterations_effective=rep.iterations_effective, max_residual_rms=rep.max_residual_rms,
                                iterations_sum=rep.iterations_sum, breakdown_fallbacks=rep.breakdown_fallbacks,
                                n_groups=len(rep.per_block_iterations)))
    shards = [None] * world
    dist.all_gather_object(shards, (np.asarray(rep.per_cell_x), rep.per_block_iterations, rep.per_block_flags))
    if rank == 0:
        np.save(out_path, np.array([merged, shards], dtype=object), allow_pickle=True)
    s.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 6])
def test_two_gpu_ranks_equal_single_run(solver, m156, tmp_path, k):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cells = 1003
    out = str(tmp_path / "out.npy")
    mp.start_processes(_rank_worker, args=(2, port, cells, k, out), nprocs=2, start_method="spawn")
    merged, shards = np.load(out, allow_pickle=True)
    v, b = m156.newton_batch(0, cells, cells, REGIME_P.h)
    whole = solver.run_strategy(BatchedSystem(156, cells, m156.row_ptr, m156.col_idx, v, b),
                                StrategyConfig(Strategy.BlockCells, k), DeviceSpec(), REGIME_P.tol, 200, 1,
                                Algo.BICGSTAB_JACOBI)
    np.testing.assert_array_equal(of.bits(np.concatenate([s[0] for s in shards])),
                                  of.bits(np.asarray(whole.per_cell_x)))
    np.testing.assert_array_equal(np.concatenate([s[1] for s in shards]), whole.per_block_iterations)
    np.testing.assert_array_equal(np.concatenate([s[2] for s in shards]), whole.per_block_flags)
    assert merged["iterations_sum"] == whole.iterations_sum
    assert merged["iterations_effective"] == whole.iterations_effective
    assert merged["breakdown_fallbacks"] == whole.breakdown_fallbacks
    assert of.bits(merged["max_residual_rms"]) == of.bits(whole.max_residual_rms)
