"""Device-resident backward-Euler simulation: the reference's run_simulation
(simulate.hpp:76-78, simulate.cpp:72-178) over bc_simulate
(include/blockcells_b200.h), SURVEY.md §8f rank 3.

Same names, fields and error behaviour as simulate.hpp: ``SimulationConfig``,
``StepStats``, ``SimulationResult``, ``run_simulation`` (raises ``ValueError``
for the reference's std::invalid_argument and ``SolverAbort`` with ``.step``
for a non-finite state).  The states, the assembled Newton systems, the
solver's vectors and the update stay in HBM for the whole run; per Newton
iteration only |dy|_inf and |y|_inf (and per step the clip count) reach the
host.  The mechanism is a ``workload.Mechanism`` (generate_mechanism(s, r,
seed) plus its evaluator tables); rate constants per cell are computed on the
host with pow(), as rate_constants does (mechanism.cpp:221-233).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native
from .solver import Algo, DeviceSpec, Solver, Strategy, StrategyConfig, _raise
from .workload import IDEAL, REALISTIC, Mechanism  # noqa: F401


class SolverAbort(RuntimeError):
    """simulate.hpp:15-19: a concentration went non-finite at ``step``."""

    def __init__(self, step: int, what: str):
        super().__init__(what)
        self.step = step


@dataclass
class LinearSolverChoice:
    """simulate.hpp:33-36 (+ the algorithm selector of SURVEY.md §8b)."""
    use_direct_reference: bool = False
    strategy: StrategyConfig = field(default_factory=lambda: StrategyConfig(Strategy.OneCell))
    algo: Algo = Algo.BICG


@dataclass
class SimulationConfig:
    """simulate.hpp:39-55."""
    cells: int = 1
    mode: int = IDEAL
    steps: int = 720
    dt_seconds: float = 120.0
    tol: float = 1e-30
    max_iter: int = 1000
    worker_count: int = 1
    solver: LinearSolverChoice = field(default_factory=LinearSolverChoice)
    device: DeviceSpec = field(default_factory=DeviceSpec)
    newton_rtol: float = 1e-10
    max_newton_iterations: int = 10


@dataclass
class StepStats:
    """simulate.hpp:59-68."""
    step: int = 0
    newton_iterations: int = 0
    iterations_effective: int = 0
    iterations_sum: int = 0
    max_residual_rms: float = 0.0
    wall_time_ns: int = 0
    breakdown_fallbacks: int = 0
    clip_events: int = 0


@dataclass
class SimulationResult:
    """simulate.hpp:70-73; final_states is (cells, species)."""
    per_step: List[StepStats] = field(default_factory=list)
    final_states: Optional[np.ndarray] = None


def default_initial_states(cells: int, species: int) -> np.ndarray:
    """simulate.cpp:66-70: every species at 1.0."""
    return np.ones((cells, species), np.float64)


def _tables(mech: Mechanism):
    prog = mech.stamp_program()
    nstamps = int(prog["stamp_ptr"][-1])
    arrs = dict(row_ptr=np.ascontiguousarray(mech.row_ptr, np.int32),
                col_idx=np.ascontiguousarray(mech.col_idx, np.int32), **prog)
    t = _native.MechTables()
    t.species, t.reactions, t.nnz, t.stamps = mech.species, mech.reactions, mech.nnz, nstamps
    for k, a in arrs.items():
        setattr(t, k, a.ctypes.data)
    return t, arrs  # keep the arrays alive while t is used


def run_simulation(mech: Mechanism, config: SimulationConfig, initial_states=None,
                   solver: Optional[Solver] = None, stream: Optional[int] = None) -> SimulationResult:
    """simulate.cpp:72-178 on the GPU.  initial_states: (cells, species)
    array (numpy or a CUDA tensor; default all ones); a CUDA tensor is
    advanced in place and returned as final_states."""
    if config.cells == 0:
        raise ValueError("run_simulation: cells must be >= 1")
    if not config.dt_seconds > 0.0:
        raise ValueError("run_simulation: dt must be positive")
    states = default_initial_states(config.cells, mech.species) if initial_states is None else initial_states
    if tuple(states.shape) != (config.cells, mech.species):
        raise ValueError("run_simulation: one initial state per cell" if states.shape[0] != config.cells
                         else "run_simulation: state dimension mismatch")
    on_device = hasattr(states, "is_cuda") and states.is_cuda
    if on_device:
        if not states.is_contiguous():
            raise ValueError("run_simulation: device states must be contiguous")
        out = states
    else:
        out = np.array(states, dtype=np.float64, order="C", copy=True)
    solver = solver or _default()
    rates = mech.rate_constants(0, config.cells, config.cells, config.mode)
    tabs, keep = _tables(mech)
    prm = _native.SimParams()
    prm.cells, prm.steps, prm.dt_seconds = config.cells, config.steps, float(config.dt_seconds)
    prm.tol, prm.max_iter = float(config.tol), int(config.max_iter)
    prm.strategy = int(config.solver.strategy.kind)
    prm.algo = int(config.solver.algo)
    k = config.solver.strategy.cells_per_block
    prm.cells_per_block = 0 if k is None else int(k)
    prm.max_threads_per_block = int(config.device.max_threads_per_block)
    prm.use_direct_reference = 1 if config.solver.use_direct_reference else 0
    prm.newton_rtol, prm.max_newton_iterations = float(config.newton_rtol), int(config.max_newton_iterations)
    prm.stream = C.c_void_p(stream) if stream else None
    stats = (_native.StepStatsC * max(1, config.steps))()
    abort = C.c_int64(-1)
    ptr = C.c_void_p(out.data_ptr()) if on_device else C.c_void_p(out.ctypes.data)
    st = _native.b200().bc_simulate(solver._ctx, C.byref(prm), C.byref(tabs), C.c_void_p(rates.ctypes.data), ptr,
                                    stats, C.byref(abort))
    del keep
    if st == -8:
        raise SolverAbort(int(abort.value), _native.b200().bc_last_error(solver._ctx).decode())
    _raise(solver._ctx, st)
    per_step = [StepStats(*(getattr(stats[i], f) for f, _ in _native.StepStatsC._fields_))
                for i in range(config.steps)]
    return SimulationResult(per_step=per_step, final_states=out)


_solver = None


def _default() -> Solver:
    global _solver
    if _solver is None:
        _solver = Solver(0)
    return _solver
