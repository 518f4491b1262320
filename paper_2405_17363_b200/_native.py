"""ctypes bindings of the in-tree native libraries.

``libbc_b200.so`` (sm_100a kernels + C ABI, include/blockcells_b200.h) and
``libbc_workload.so`` (synthetic workload generator, include/blockcells_workload.h)
are built in-tree by ``__graft_entry__.build()`` / ``make -C
paper_2405_17363_b200/csrc``.  There is deliberately no fallback: if the
library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_B200 = os.path.join(_HERE, "libbc_b200.so")
LIB_WORKLOAD = os.path.join(_HERE, "libbc_workload.so")

_c_p = C.c_void_p
_i32, _i64, _u64, _f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class SolveParams(C.Structure):
    _fields_ = [
        ("strategy", _i32), ("algo", _i32), ("cells_per_block", _i64), ("cells", _i64),
        ("tol", _f64), ("max_iter", _i64), ("max_threads_per_block", _i64),
        ("stream", _c_p), ("options", _i32), ("reserved", _i32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("n_groups", _i64), ("iterations_effective", _i64), ("iterations_sum", _i64),
        ("max_residual_rms", _f64), ("breakdown_fallbacks", _i64), ("cells_per_block", _f64),
        ("device_ms", _f64), ("kernel_launches", _i64), ("kernels", _i32), ("reserved", _i32),
        ("model_spmv_wavefronts", _f64),
    ]


class Outcome(C.Structure):
    _fields_ = [("iterations", _i64), ("final_residual_rms", _f64),
                ("converged", _i32), ("breakdown", _i32)]


class SimParams(C.Structure):  # bc_sim_params (SimulationConfig)
    _fields_ = [
        ("cells", _i64), ("steps", _i64), ("dt_seconds", _f64), ("tol", _f64), ("max_iter", _i64),
        ("strategy", _i32), ("algo", _i32), ("cells_per_block", _i64), ("max_threads_per_block", _i64),
        ("use_direct_reference", _i32), ("reserved", _i32), ("newton_rtol", _f64),
        ("max_newton_iterations", _i64), ("stream", _c_p),
    ]


class StepStatsC(C.Structure):  # bc_step_stats (StepStats)
    _fields_ = [
        ("step", _i64), ("newton_iterations", _i64), ("iterations_effective", _i64), ("iterations_sum", _i64),
        ("max_residual_rms", _f64), ("wall_time_ns", _i64), ("breakdown_fallbacks", _i64),
        ("clip_events", _i64),
    ]


class MechTables(C.Structure):  # bc_mechanism_tables
    _fields_ = [("species", _i32), ("reactions", _i32), ("nnz", _i32), ("stamps", _i32)] + [
        (n, _c_p) for n in ("row_ptr", "col_idx", "stamp_ptr", "stamp_slot", "stamp_other", "stamp_sign",
                            "reactant_ptr", "reactants", "product_ptr", "products", "diag_slot")]


def _load(path: str, what: str) -> C.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(
            f"{what} not built: {path} is missing. Run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2405_17363_b200/csrc` (no CPU fallback exists).")
    return C.CDLL(path)


_b200 = None
_wl = None


def b200() -> C.CDLL:
    global _b200
    if _b200 is None:
        lib = _load(LIB_B200, "libbc_b200.so (CUDA sm_100a solver)")
        lib.bc_ctx_create.argtypes = [C.c_int, C.POINTER(_c_p)]
        lib.bc_ctx_destroy.argtypes = [_c_p]
        lib.bc_ctx_destroy.restype = None
        lib.bc_last_error.argtypes = [_c_p]
        lib.bc_last_error.restype = C.c_char_p
        lib.bc_set_pattern.argtypes = [_c_p, _i32, _c_p, _c_p]
        lib.bc_plan.argtypes = [_i32, C.POINTER(SolveParams), C.POINTER(_i64), C.POINTER(_f64)]
        lib.bc_schedule_export.argtypes = [_i32, _c_p, _c_p, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]
        lib.bc_tmem_schedule_export.argtypes = [_i32, _c_p, _c_p, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p]
        lib.bc_solve.argtypes = [_c_p, C.POINTER(SolveParams), _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                 C.POINTER(Report)]
        lib.bc_bicg_solve.argtypes = [_c_p, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _f64, _i64,
                                      _i64, _c_p, _c_p, C.POINTER(Outcome)]
        lib.bc_kernel_launches.argtypes = [_c_p]
        lib.bc_kernel_launches.restype = _i64
        lib.bc_newton_assemble.argtypes = [_c_p, _i64, _i32, _i32, _i32] + [_c_p] * 10 + [
            _f64, _c_p, _c_p, _c_p, _c_p, _c_p]
        lib.bc_simulate.argtypes = [_c_p, C.POINTER(SimParams), C.POINTER(MechTables), _c_p, _c_p, _c_p,
                                    C.POINTER(_i64)]
        lib.bc_ctx_pattern_info.argtypes = [_c_p, _c_p]
        lib.bc_latency_schedule_export.argtypes = [_i32, _c_p, _c_p, _i32, _i32, _i32] + [_c_p] * 8
        lib.bc_devset_create.argtypes = [C.c_int, _c_p, C.POINTER(_c_p)]
        lib.bc_devset_destroy.argtypes = [_c_p]
        lib.bc_devset_destroy.restype = None
        lib.bc_devset_size.argtypes = [_c_p]
        lib.bc_devset_last_error.argtypes = [_c_p]
        lib.bc_devset_last_error.restype = C.c_char_p
        lib.bc_devset_set_pattern.argtypes = [_c_p, _i32, _c_p, _c_p]
        lib.bc_devset_solve.argtypes = lib.bc_solve.argtypes
        lib.bc_host_alloc.argtypes = [_u64, C.POINTER(_c_p)]
        lib.bc_host_free.argtypes = [_c_p]
        lib.bc_host_free.restype = None
        _b200 = lib
    return _b200


def workload() -> C.CDLL:
    global _wl
    if _wl is None:
        lib = _load(LIB_WORKLOAD, "libbc_workload.so (workload generator)")
        lib.bcw_mechanism_create.argtypes = [_i64, _i64, _u64, C.POINTER(_c_p)]
        lib.bcw_mechanism_destroy.argtypes = [_c_p]
        lib.bcw_mechanism_destroy.restype = None
        for f in ("bcw_species", "bcw_reactions", "bcw_nnz", "bcw_stamp_count"):
            getattr(lib, f).argtypes = [_c_p]
            getattr(lib, f).restype = _i64
        lib.bcw_pattern.argtypes = [_c_p, _c_p, _c_p]
        lib.bcw_newton_batch.argtypes = [_c_p, _i64, _i64, _i64, C.c_int, _f64, _c_p, _c_p, _c_p, _c_p,
                                         C.c_int]
        lib.bcw_rate_constants.argtypes = [_c_p, _i64, _i64, _i64, C.c_int, _c_p, C.c_int]
        lib.bcw_stamp_program.argtypes = [_c_p] * 10
        _wl = lib
    return _wl
