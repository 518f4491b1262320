"""The Python mirror's argument checks (the reference throws
std::invalid_argument for the same contract violations), and the
pattern-cache regression the advisor found: a context whose pattern was
replaced by bc_simulate must not solve the next batch with it."""
from __future__ import annotations

import numpy as np
import pytest

from fixtures import random_batch
from paper_2405_17363_b200 import Algo, BatchedSystem, DeviceSpec, Mechanism, Strategy, StrategyConfig


def test_device_spec_check_mirrors_reference():
    DeviceSpec().check()
    with pytest.raises(ValueError):
        DeviceSpec(max_threads_per_block=0).check()
    with pytest.raises(ValueError):
        DeviceSpec(warp_size=-1).check()
    with pytest.raises(ValueError):
        DeviceSpec(max_threads_per_block=4096, max_threads_per_sm=2048).check()


def test_batched_system_rejects_wrong_dtype_and_shape():
    rng = np.random.default_rng(0)
    rp, ci, v, b = random_batch(rng, 3, 8)
    BatchedSystem(8, 3, rp, ci, v, b).check()
    with pytest.raises(ValueError):
        BatchedSystem(8, 3, rp, ci, v.astype(np.float32), b).check()
    with pytest.raises(ValueError):
        BatchedSystem(8, 3, rp, ci, v, b.astype(np.int64)).check()
    with pytest.raises(ValueError):
        BatchedSystem(8, 3, rp, ci, v[:2], b).check()
    with pytest.raises(ValueError):
        BatchedSystem(8, 3, rp, ci, v, b[:, :7]).check()


def test_newton_batch_rejects_bad_output_buffers():
    m = Mechanism(24, 72, 1)
    m.newton_batch(0, 4, 4, 1.0)
    with pytest.raises(ValueError):
        m.newton_batch(0, 4, 4, 1.0, values=np.empty((4, m.nnz), np.float32))
    with pytest.raises(ValueError):
        m.newton_batch(0, 4, 4, 1.0, rhs=np.empty((3, m.species)))
    with pytest.raises(ValueError):
        m.newton_batch(0, 4, 4, 1.0, y=np.ones((4, m.species + 1)))


@pytest.mark.gpu
def test_solver_rejects_bad_outputs_and_devices(solver):
    import torch
    rng = np.random.default_rng(1)
    rp, ci, v, b = random_batch(rng, 5, 12)
    sysm = BatchedSystem(12, 5, rp, ci, v, b)
    cfg = StrategyConfig(Strategy.BlockCells, 1)
    with pytest.raises(ValueError):
        solver.run_strategy(sysm, cfg, DeviceSpec(), 1e-10, 100, x_out=np.empty((5, 11)))
    with pytest.raises(ValueError):
        solver.run_strategy(sysm, cfg, DeviceSpec(), 1e-10, 100, x_out=np.empty((5, 12), np.float32))
    with pytest.raises(ValueError):
        solver.run_strategy(sysm, cfg, DeviceSpec(max_threads_per_block=0), 1e-10, 100)
    with pytest.raises(ValueError):
        solver.run_strategy(BatchedSystem(12, 5, rp, ci, torch.from_numpy(v).float().cuda(),
                                          torch.from_numpy(b).cuda()), cfg, DeviceSpec(), 1e-10, 100)
    rep = solver.run_strategy(sysm, cfg, DeviceSpec(), 1e-10, 100, x_out=np.empty((5, 12)))
    assert rep.per_cell_x.shape == (5, 12)


@pytest.mark.gpu
def test_pattern_switch_between_run_strategy_and_simulation(solver):
    """run_strategy(A), run_simulation (installs mechanism B's pattern on the
    same context), run_strategy(A) again: the second solve is A's, bit for
    bit (a caller-side pattern cache went stale here)."""
    from paper_2405_17363_b200 import simulate as sim
    rng = np.random.default_rng(2)
    rp, ci, v, b = random_batch(rng, 40, 30, 0.2)
    sysm = BatchedSystem(30, 40, rp, ci, v, b)
    cfg = StrategyConfig(Strategy.BlockCells, 1)
    first = solver.run_strategy(sysm, cfg, DeviceSpec(), 1e-12, 300, algo=Algo.BICGSTAB_JACOBI)
    mech = Mechanism(24, 72, 3)
    config = sim.SimulationConfig(cells=16, steps=1, dt_seconds=1.0, tol=1e-10, max_iter=100)
    sim.run_simulation(mech, config, solver=solver)
    again = solver.run_strategy(sysm, cfg, DeviceSpec(), 1e-12, 300, algo=Algo.BICGSTAB_JACOBI)
    np.testing.assert_array_equal(np.asarray(first.per_cell_x).view(np.uint64),
                                  np.asarray(again.per_cell_x).view(np.uint64))
    np.testing.assert_array_equal(first.per_block_iterations, again.per_block_iterations)
