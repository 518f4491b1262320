"""CPU, world_size 2 (gloo): the multi-GPU path's host logic.  Each rank
generates its shard of a global batch (global cell conditions), solves it
(here with the CPU oracle standing in for the per-GPU solve, which is
bit-identical to it -- tests/test_gpu_parity.py), and the merged results must
equal the single-process solve of the whole batch bit for bit."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ffi as of
from paper_2405_17363_b200 import Mechanism
from paper_2405_17363_b200.sharding import group_offset, merge_reports, shard_range


def test_shard_range_partitions_at_group_boundaries():
    for cells in (1, 7, 100, 1001):
        for k in (1, 3, 6):
            for world in (1, 2, 3, 8):
                covered, groups = [], 0
                for rank in range(world):
                    first, count = shard_range(cells, k, rank, world)
                    assert first % k == 0
                    assert group_offset(cells, k, rank, world) == groups
                    covered.extend(range(first, first + count))
                    groups += count // k + (1 if count % k else 0)
                assert covered == list(range(cells))
                assert groups == cells // k + (1 if cells % k else 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cells, k, h, tol, max_iter, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = Mechanism(40, 120, 3)
    first, count = shard_range(cells, k, rank, world)
    v, b = m.newton_batch(first, count, cells, h)  # global cell conditions
    st, res = of.orc_solve_batch(2, 1, k, m.row_ptr, m.col_idx, v, b, tol, max_iter)
    assert st == 0
    r = res.report
    merged = merge_reports(dict(iterations_effective=r.iterations_effective, max_residual_rms=r.max_residual_rms,
                                iterations_sum=r.iterations_sum, breakdown_fallbacks=r.breakdown_fallbacks,
                                n_groups=r.n_groups))
    shards = [None] * world
    dist.all_gather_object(shards, (first, res.x, res.iters, res.rms, res.flags))
    if rank == 0:
        np.save(out_path, np.array([merged, shards], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 4])
def test_two_rank_shards_equal_single_run(tmp_path, k):
    cells, h, tol, max_iter = 37, 120.0, 1e-30, 60
    out = str(tmp_path / "out.npy")
    mp.start_processes(_worker, args=(2, _free_port(), cells, k, h, tol, max_iter, out), nprocs=2,
                       start_method="spawn")
    merged, shards = np.load(out, allow_pickle=True)
    m = Mechanism(40, 120, 3)
    v, b = m.newton_batch(0, cells, cells, h)
    st, whole = of.orc_solve_batch(2, 1, k, m.row_ptr, m.col_idx, v, b, tol, max_iter)
    assert st == 0
    x = np.concatenate([s[1] for s in shards])
    iters = np.concatenate([s[2] for s in shards])
    np.testing.assert_array_equal(of.bits(x), of.bits(whole.x))
    np.testing.assert_array_equal(iters, whole.iters)
    np.testing.assert_array_equal(of.bits(np.concatenate([s[3] for s in shards])), of.bits(whole.rms))
    w = whole.report
    assert merged["iterations_effective"] == w.iterations_effective
    assert merged["iterations_sum"] == w.iterations_sum
    assert merged["breakdown_fallbacks"] == w.breakdown_fallbacks
    assert merged["n_groups"] == w.n_groups
    assert of.bits(merged["max_residual_rms"]) == of.bits(w.max_residual_rms)
