"""Host-side mirror of the reference's solver API (strategies.hpp / bicg.hpp).

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/core/include/blockcells/strategies.hpp:15-90,
bicg.hpp:25-48, exec_model.hpp:14-43), implemented over the C ABI of
``libbc_b200.so``.  All arithmetic runs in the sm_100a kernels; this module
only marshals arrays.  Arrays may be numpy (host) or CUDA torch tensors
(device-resident, no copies).
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from ._native import Outcome, Report, SolveParams


class InvalidGrouping(ValueError):
    """exec_model.hpp:19-21 -- requested cells-per-block does not fit."""


class UnsupportedMechanism(ValueError):
    """exec_model.hpp:14-16 -- species exceed the block's thread budget."""


class SingularMatrix(RuntimeError):
    """dense_lu.hpp:12-14 -- zero pivot in the LU fallback."""


class CudaError(RuntimeError):
    pass


class Strategy(enum.IntEnum):
    OneCell = 0
    MultiCells = 1
    BlockCells = 2
    ThreadPerCell = 3  # comparison baseline (one thread per cell)


class Algo(enum.IntEnum):
    BICG = 0
    BICGSTAB_JACOBI = 1


FLAG_CONVERGED, FLAG_BREAKDOWN, FLAG_FELL_BACK = 1, 2, 4


@dataclass
class DeviceSpec:
    """exec_model.hpp:31-43.  Only max_threads_per_block changes results
    (grouping k and the Multi-cells reduction width); the other limits only
    fed the reference's analytic occupancy model."""
    max_threads_per_block: int = 1024
    warp_size: int = 32
    max_warps_per_sm: int = 64
    max_blocks_per_sm: int = 32
    max_threads_per_sm: int = 2048
    shared_mem_per_sm: int = 96 * 1024
    shared_slot_bytes: int = 8

    def check(self) -> None:
        """DeviceSpec::check (exec_model.hpp:40-42): every limit positive and
        max_threads_per_block <= max_threads_per_sm, std::invalid_argument there."""
        for f in ("max_threads_per_block", "warp_size", "max_warps_per_sm", "max_blocks_per_sm",
                  "max_threads_per_sm", "shared_mem_per_sm", "shared_slot_bytes"):
            if int(getattr(self, f)) <= 0:
                raise ValueError(f"device spec: {f} must be positive")
        if self.max_threads_per_block > self.max_threads_per_sm:
            raise ValueError("device spec: max_threads_per_block exceeds max_threads_per_sm")


@dataclass
class StrategyConfig:
    kind: Strategy = Strategy.OneCell
    cells_per_block: Optional[int] = None


@dataclass
class BatchedSystem:
    """strategies.hpp:15-23 with the shared pattern stored once:
    values[c] is per_cell_matrices[c].values, rhs[c] is per_cell_rhs[c]."""
    species: int
    cells: int
    row_ptr: np.ndarray   # int32, species+1
    col_idx: np.ndarray   # int32, nnz
    values: object        # (cells, nnz) float64: numpy or CUDA tensor
    rhs: object           # (cells, species) float64: numpy or CUDA tensor

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def check(self) -> None:
        """strategies.cpp:91-107 (the shared pattern holds by construction)."""
        if self.cells == 0:
            raise ValueError("batched system: no cells")
        if self.species == 0:
            raise ValueError("batched system: no species")
        if tuple(_shape(self.values)) != (self.cells, self.nnz) or tuple(_shape(self.rhs)) != (self.cells, self.species):
            raise ValueError("batched system: per-cell arrays mismatch")
        _check_f64(self.values, "values")
        _check_f64(self.rhs, "rhs")
        if _is_torch_cuda(self.values) != _is_torch_cuda(self.rhs) or (
                _is_torch_cuda(self.values) and self.values.device != self.rhs.device):
            raise ValueError("batched system: values and rhs must live on the same device")


@dataclass
class SolveReport:
    """strategies.hpp:35-48 plus per-group residual/flags and device time."""
    strategy: Strategy = Strategy.OneCell
    cells_per_block: float = 1.0
    iterations_effective: int = 0
    iterations_sum: int = 0
    per_block_iterations: object = None  # (groups,) int64 array: strategies.hpp:40's vector
    max_residual_rms: float = 0.0
    wall_time_ns: int = 0
    breakdown_fallbacks: int = 0
    per_cell_x: object = None            # (cells, species)
    per_block_residual_rms: object = None
    per_block_flags: object = None
    device_ms: float = 0.0
    kernel_launches: int = 0
    kernels: int = 0                     # KERNEL_* bits of the kernels launched
    model_spmv_wavefronts: float = 0.0   # planner's modelled shared wavefronts per group-iteration (TMEM kernel)


# bc_report.kernels bits (include/blockcells_b200.h)
KERNEL_TMEM, KERNEL_BLOCK, KERNEL_MULTI, KERNEL_THREAD, KERNEL_LU, KERNEL_LATENCY = 1, 2, 4, 8, 16, 32


@dataclass
class SolveOutcome:
    """bicg.hpp:25-31."""
    x: np.ndarray
    iterations: int = 0
    final_residual_rms: float = 0.0
    converged: bool = False
    breakdown: bool = False


@dataclass
class ReductionPlan:
    """reduction.hpp:25-37."""
    block_ranges: List[Tuple[int, int]]
    host_stage: bool = False

    @staticmethod
    def single_block(n: int) -> "ReductionPlan":
        return ReductionPlan([(0, n)], False)


def _shape(a):
    return tuple(a.shape)


def _is_torch_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _check_f64(a, name: str) -> None:
    """The C ABI reads 8 bytes per element: anything but float64 would be
    read past its end."""
    dt = getattr(a, "dtype", None)
    if hasattr(a, "data_ptr"):  # torch tensor
        import torch
        ok = dt == torch.float64
    else:
        ok = dt == np.float64
    if not ok:
        raise ValueError(f"{name} must be float64 (got {dt})")


def _check_out(x, shape, like, name: str, device: int) -> None:
    """A caller-supplied output: exact shape, float64, contiguous, and on
    the solver's GPU when it is a CUDA tensor."""
    if tuple(_shape(x)) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)} (got {tuple(_shape(x))})")
    _check_f64(x, name)
    if _is_torch_cuda(x) and device >= 0 and x.device.index != device:
        raise ValueError(f"{name} is on {x.device}, the solver runs on cuda:{device}")


def _ptr(a):
    if a is None:
        return None
    if _is_torch_cuda(a) or (hasattr(a, "data_ptr") and hasattr(a, "is_pinned")):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return C.c_void_p(a.ctypes.data)


def _raise(ctx, code: int) -> None:
    if code == 0:
        return
    msg = _native.b200().bc_last_error(ctx).decode()
    if code == -2:
        raise InvalidGrouping(msg)
    if code == -3:
        raise UnsupportedMechanism(msg)
    if code == -4:
        raise SingularMatrix(msg)
    if code in (-1, -6):
        raise ValueError(msg)
    if code == -7:
        raise MemoryError(msg)
    raise CudaError(f"{msg} (status {code})")


class Solver:
    """One CUDA context (bc_ctx) bound to one GPU."""

    def __init__(self, device: int = 0):
        lib = _native.b200()
        self._ctx = C.c_void_p()
        st = lib.bc_ctx_create(int(device), C.byref(self._ctx))
        if st != 0:
            raise CudaError(f"bc_ctx_create(device={device}) failed with status {st}")
        self.device = device

    def close(self) -> None:
        if self._ctx:
            _native.b200().bc_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return int(_native.b200().bc_kernel_launches(self._ctx))

    def set_pattern(self, species: int, row_ptr: np.ndarray, col_idx: np.ndarray) -> None:
        """bc_set_pattern keeps the context's schedules when the pattern is the
        one already installed (it compares against its own state, so nothing
        is cached here that bc_simulate could make stale)."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        if rp.ndim != 1 or rp.shape[0] != int(species) + 1 or ci.ndim != 1 or ci.shape[0] < int(rp[-1]):
            raise ValueError("csr: row_ptr/col_idx shape does not match species")
        _raise(self._ctx, _native.b200().bc_set_pattern(self._ctx, int(species), _ptr(rp), _ptr(ci)))

    def group_count(self, system: BatchedSystem, config: StrategyConfig, device: DeviceSpec = DeviceSpec()) -> Tuple[int, float]:
        device.check()
        self.set_pattern(system.species, system.row_ptr, system.col_idx)
        prm = self._params(system, config, Algo.BICG, device, 1.0, 1, None, False)
        ng, cpb = C.c_int64(), C.c_double()
        _raise(self._ctx, _native.b200().bc_plan(int(system.species), C.byref(prm), C.byref(ng), C.byref(cpb)))
        return int(ng.value), float(cpb.value)

    @staticmethod
    def _params(system, config, algo, device, tol, max_iter, stream, timing) -> SolveParams:
        prm = SolveParams()
        prm.strategy = int(config.kind)
        prm.algo = int(algo)
        if config.cells_per_block is None:
            prm.cells_per_block = 0
        else:
            if int(config.cells_per_block) < 1:
                raise ValueError("plan_kernel: cells per block must be >= 1")
            prm.cells_per_block = int(config.cells_per_block)
        prm.cells = int(system.cells)
        prm.tol = float(tol)
        prm.max_iter = int(max_iter)
        prm.max_threads_per_block = int(device.max_threads_per_block)
        prm.stream = C.c_void_p(stream) if stream else None
        prm.options = 1 if timing else 0
        return prm

    def run_strategy(self, system: BatchedSystem, config: StrategyConfig, device: DeviceSpec = DeviceSpec(),
                     tol: float = 1e-30, max_iter: int = 1000, worker_count: int = 1,
                     algo: Algo = Algo.BICG, stream: Optional[int] = None, timing: bool = False,
                     x_out=None) -> SolveReport:
        """strategies.cpp:251-264.  worker_count is accepted for API parity; the
        GPU result is independent of it, as the reference's is."""
        system.check()
        device.check()
        if max_iter < 1:
            raise ValueError("bicg: max_iter must be >= 1")
        if _is_torch_cuda(system.values) and system.values.device.index != self.device:
            raise ValueError(f"batched system is on {system.values.device}, the solver runs on cuda:{self.device}")
        if x_out is not None:
            _check_out(x_out, (system.cells, system.species), system.values, "x_out", self.device)
        self.set_pattern(system.species, system.row_ptr, system.col_idx)
        prm = self._params(system, config, algo, device, tol, max_iter, stream, timing)
        lib = _native.b200()
        ng, cpb = C.c_int64(), C.c_double()
        _raise(self._ctx, lib.bc_plan(int(system.species), C.byref(prm), C.byref(ng), C.byref(cpb)))
        ng = int(ng.value)
        on_device = _is_torch_cuda(system.values)
        if x_out is None:
            if on_device:
                import torch
                x_out = torch.empty((system.cells, system.species), dtype=torch.float64, device=system.values.device)
            else:
                x_out = np.empty((system.cells, system.species), dtype=np.float64)
        iters = np.empty(ng, np.int32)
        rms = np.empty(ng, np.float64)
        flags = np.empty(ng, np.uint8)
        rep = Report()
        t0 = time.perf_counter_ns()
        st = lib.bc_solve(self._ctx, C.byref(prm), _ptr(system.values), _ptr(system.rhs), _ptr(x_out),
                          _ptr(iters), _ptr(rms), _ptr(flags), C.byref(rep))
        wall = time.perf_counter_ns() - t0
        _raise(self._ctx, st)
        return SolveReport(
            strategy=Strategy(config.kind), cells_per_block=float(rep.cells_per_block),
            iterations_effective=int(rep.iterations_effective), iterations_sum=int(rep.iterations_sum),
            per_block_iterations=iters.astype(np.int64), max_residual_rms=float(rep.max_residual_rms),
            wall_time_ns=int(wall), breakdown_fallbacks=int(rep.breakdown_fallbacks), per_cell_x=x_out,
            per_block_residual_rms=rms, per_block_flags=flags, device_ms=float(rep.device_ms),
            kernel_launches=int(rep.kernel_launches), kernels=int(rep.kernels),
            model_spmv_wavefronts=float(rep.model_spmv_wavefronts))

    # strategies.hpp:60-77
    def solve_one_cell(self, system, tol, max_iter, device: DeviceSpec = DeviceSpec(), algo=Algo.BICG, **kw):
        return self.run_strategy(system, StrategyConfig(Strategy.OneCell), device, tol, max_iter, 1, algo, **kw)

    def solve_multi_cells(self, system, device: DeviceSpec, tol, max_iter, algo=Algo.BICG, **kw):
        return self.run_strategy(system, StrategyConfig(Strategy.MultiCells), device, tol, max_iter, 1, algo, **kw)

    def solve_block_cells(self, system, cells_per_block, device: DeviceSpec, tol, max_iter, worker_count=1,
                          algo=Algo.BICG, **kw):
        return self.run_strategy(system, StrategyConfig(Strategy.BlockCells, cells_per_block), device, tol,
                                 max_iter, worker_count, algo, **kw)

    def bicg_solve(self, n: int, row_ptr, col_idx, vals, b, x0, tol: float, max_iter: int,
                   plan: Optional[ReductionPlan] = None, algo: Algo = Algo.BICG) -> SolveOutcome:
        """bicg.hpp:42-48 on one system with its own pattern."""
        plan = plan or ReductionPlan.single_block(n)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        va = np.ascontiguousarray(vals, dtype=np.float64)
        bb = np.ascontiguousarray(b, dtype=np.float64)
        x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        ranges = np.ascontiguousarray(np.array(plan.block_ranges, dtype=np.int64).reshape(-1))
        x = np.empty(n, np.float64)
        out = Outcome()
        st = _native.b200().bc_bicg_solve(self._ctx, int(algo), int(n), _ptr(rp), _ptr(ci), _ptr(va), _ptr(bb),
                                          _ptr(x0a), float(tol), int(max_iter), len(plan.block_ranges),
                                          _ptr(ranges), _ptr(x), C.byref(out))
        _raise(self._ctx, st)
        return SolveOutcome(x, int(out.iterations), float(out.final_residual_rms), bool(out.converged),
                            bool(out.breakdown))


class DeviceSet:
    """The drop-in API over several GPUs of one box (bc_devset, SURVEY.md
    §8e): contiguous group-aligned shards, one host thread per GPU, report
    merged in group order -- bit-identical to one Solver.  A device may be
    listed twice (two contexts on one GPU).  Arrays: host memory (numpy;
    pinned buffers stream into the solve)."""

    def __init__(self, devices):
        lib = _native.b200()
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        self._set = C.c_void_p()
        st = lib.bc_devset_create(len(devices), devs, C.byref(self._set))
        if st != 0:
            raise CudaError(f"bc_devset_create({list(devices)}) failed with status {st}")
        self.devices = list(devices)

    def close(self) -> None:
        if self._set:
            _native.b200().bc_devset_destroy(self._set)
            self._set = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, code):
        if code == 0:
            return
        msg = _native.b200().bc_devset_last_error(self._set).decode()
        exc = {-2: InvalidGrouping, -3: UnsupportedMechanism, -4: SingularMatrix, -1: ValueError,
               -6: ValueError, -7: MemoryError}.get(code)
        raise (exc or CudaError)(msg if exc else f"{msg} (status {code})")

    def run_strategy(self, system: BatchedSystem, config: StrategyConfig, device: DeviceSpec = DeviceSpec(),
                     tol: float = 1e-30, max_iter: int = 1000, worker_count: int = 1,
                     algo: Algo = Algo.BICG, timing: bool = False, x_out=None) -> SolveReport:
        system.check()
        device.check()
        if max_iter < 1:
            raise ValueError("bicg: max_iter must be >= 1")
        if x_out is None:
            x_out = np.empty((system.cells, system.species), dtype=np.float64)
        else:
            _check_out(x_out, (system.cells, system.species), system.values, "x_out", -1)
        lib = _native.b200()
        rp = np.ascontiguousarray(system.row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(system.col_idx, dtype=np.int32)
        self._raise(lib.bc_devset_set_pattern(self._set, int(system.species), _ptr(rp), _ptr(ci)))
        prm = Solver._params(system, config, algo, device, tol, max_iter, None, timing)
        ng, cpb = C.c_int64(), C.c_double()
        _raise(None, lib.bc_plan(int(system.species), C.byref(prm), C.byref(ng), C.byref(cpb)))
        ng = int(ng.value)
        iters = np.empty(ng, np.int32)
        rms = np.empty(ng, np.float64)
        flags = np.empty(ng, np.uint8)
        rep = Report()
        t0 = time.perf_counter_ns()
        st = lib.bc_devset_solve(self._set, C.byref(prm), _ptr(system.values), _ptr(system.rhs), _ptr(x_out),
                                 _ptr(iters), _ptr(rms), _ptr(flags), C.byref(rep))
        wall = time.perf_counter_ns() - t0
        self._raise(st)
        return SolveReport(
            strategy=Strategy(config.kind), cells_per_block=float(rep.cells_per_block),
            iterations_effective=int(rep.iterations_effective), iterations_sum=int(rep.iterations_sum),
            per_block_iterations=iters.astype(np.int64), max_residual_rms=float(rep.max_residual_rms),
            wall_time_ns=int(wall), breakdown_fallbacks=int(rep.breakdown_fallbacks), per_cell_x=x_out,
            per_block_residual_rms=rms, per_block_flags=flags, device_ms=float(rep.device_ms),
            kernel_launches=int(rep.kernel_launches), kernels=int(rep.kernels),
            model_spmv_wavefronts=float(rep.model_spmv_wavefronts))


_default: dict = {}


def default_solver(device: int = 0) -> Solver:
    if device not in _default:
        _default[device] = Solver(device)
    return _default[device]


# Free functions with the reference's names and signatures.
def run_strategy(system, config, device=DeviceSpec(), tol=1e-30, max_iter=1000, worker_count=1,
                 algo=Algo.BICG, **kw) -> SolveReport:
    return default_solver().run_strategy(system, config, device, tol, max_iter, worker_count, algo, **kw)


def solve_one_cell(system, tol, max_iter, device=DeviceSpec(), algo=Algo.BICG, **kw) -> SolveReport:
    return default_solver().solve_one_cell(system, tol, max_iter, device, algo, **kw)


def solve_multi_cells(system, device, tol, max_iter, algo=Algo.BICG, **kw) -> SolveReport:
    return default_solver().solve_multi_cells(system, device, tol, max_iter, algo, **kw)


def solve_block_cells(system, cells_per_block, device, tol, max_iter, worker_count=1, algo=Algo.BICG,
                      **kw) -> SolveReport:
    return default_solver().solve_block_cells(system, cells_per_block, device, tol, max_iter, worker_count,
                                              algo, **kw)


def bicg_solve(n, row_ptr, col_idx, vals, b, x0, tol, max_iter, plan=None, algo=Algo.BICG) -> SolveOutcome:
    return default_solver().bicg_solve(n, row_ptr, col_idx, vals, b, x0, tol, max_iter, plan, algo)


def iteration_reduction_ratio(report_a: SolveReport, report_b: SolveReport) -> float:
    """strategies.cpp:266-273."""
    if report_a.iterations_effective == 0:
        raise ValueError("iteration_reduction_ratio: zero denominator")
    return report_b.iterations_effective / report_a.iterations_effective
