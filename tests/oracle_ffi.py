"""Test-side bindings of the checkers under oracle/ (test infrastructure only).

* ``orc``  -- oracle/liborc.so, the C restatement (bc_oracle.c)
* ``ref``  -- oracle/_ref/libbcref.so, the unmodified reference compiled from
              /root/reference sources (absent on machines without the
              reference; tests that need it skip, the golden fixtures in
              tests/golden/ cover the oracle there).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORC_PATH = os.path.join(ROOT, "oracle", "liborc.so")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libbcref.so")

_i32, _i64, _f64, _p = C.c_int32, C.c_int64, C.c_double, C.c_void_p


class OrcReport(C.Structure):
    _fields_ = [("n_groups", _i64), ("iterations_effective", _i64), ("iterations_sum", _i64),
                ("max_residual_rms", _f64), ("breakdown_fallbacks", _i64), ("cells_per_block", _f64)]


class RefReport(C.Structure):
    _fields_ = OrcReport._fields_ + [("wall_time_ns", _i64)]


class OrcOutcome(C.Structure):
    _fields_ = [("iterations", _i64), ("final_residual_rms", _f64), ("converged", _i32), ("breakdown", _i32)]


def ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


_orc = None
_ref = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_PATH):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "orc"], check=True,
                           stdout=subprocess.DEVNULL)
        lib = C.CDLL(ORC_PATH)
        lib.orc_group_count.restype = _i64
        lib.orc_group_count.argtypes = [C.c_int, _i64, _i64, _i64, _i64]
        lib.orc_solve_batch.argtypes = [C.c_int, C.c_int, _i64, _i64, _i64, _p, _p, _p, _p, _f64, _i64, _i64,
                                        _i64, _p, _p, _p, _p, C.POINTER(OrcReport)]
        for f in ("orc_bicg_solve", "orc_bicgstab_solve"):
            getattr(lib, f).argtypes = [_i64, _p, _p, _p, _p, _p, _f64, _i64, _p, _i64, _p, C.POINTER(OrcOutcome)]
        lib.orc_lu_solve_csr.argtypes = [_i64, _p, _p, _p, _p, _p]
        lib.orc_tree_reduce_in_place.restype = _f64
        lib.orc_tree_reduce_in_place.argtypes = [_p, _i64]
        lib.orc_plan_reduce.restype = _f64
        lib.orc_plan_reduce.argtypes = [_p, _i64, _p, _i64, _p, _p]
        _orc = lib
    return _orc


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_PATH)
        lib.ref_solve_batch.argtypes = [C.c_int, _i64, _i64, _i64, _p, _p, _p, _p, _f64, _i64, _i64, _i64, _p, _p,
                                        C.POINTER(RefReport)]
        lib.ref_bicg_solve.argtypes = [_i64, _p, _p, _p, _p, _p, _f64, _i64, _p, _i64, C.c_int, _p,
                                       C.POINTER(_i64), C.POINTER(_f64), C.POINTER(_i32), C.POINTER(_i32)]
        lib.ref_lu_solve.argtypes = [_i64, _p, _p, _p, _p, _p]
        lib.ref_tree_reduce.restype = _f64
        lib.ref_tree_reduce.argtypes = [_p, _i64, _i64]
        lib.ref_plan_reduce.restype = _f64
        lib.ref_plan_reduce.argtypes = [_p, _i64, _p, _i64]
        lib.ref_mechanism_pattern.argtypes = [_i64, _i64, C.c_uint64, C.POINTER(_i64), _p, _p]
        lib.ref_newton_batch.argtypes = [_i64, _i64, C.c_uint64, _i64, _i64, _i64, C.c_int, _f64, _p, _p]
        _ref = lib
    return _ref


class BatchResult:
    def __init__(self, x, iters, rms, flags, report):
        self.x, self.iters, self.rms, self.flags, self.report = x, iters, rms, flags, report


def orc_solve_batch(strategy, algo, k, row_ptr, col_idx, values, rhs, tol, max_iter, mtpb=1024, workers=1):
    species = len(row_ptr) - 1
    cells = values.shape[0]
    lib = orc()
    ng = lib.orc_group_count(strategy, cells, species, mtpb, k)
    if ng < 0:
        ng = 1
    x = np.empty((cells, species))
    it = np.zeros(ng, np.int64)
    rms = np.zeros(ng)
    fl = np.zeros(ng, np.uint8)
    rep = OrcReport()
    st = lib.orc_solve_batch(strategy, algo, k, species, cells, ptr(np.ascontiguousarray(row_ptr, np.int32)),
                             ptr(np.ascontiguousarray(col_idx, np.int32)), ptr(np.ascontiguousarray(values)),
                             ptr(np.ascontiguousarray(rhs)), tol, max_iter, mtpb, workers, ptr(x), ptr(it), ptr(rms),
                             ptr(fl), C.byref(rep))
    return st, BatchResult(x, it, rms, fl, rep)


def ref_solve_batch(strategy, k, row_ptr, col_idx, values, rhs, tol, max_iter, mtpb=1024, workers=1):
    species = len(row_ptr) - 1
    cells = values.shape[0]
    ng = orc().orc_group_count(strategy, cells, species, mtpb, k)
    if ng < 0:
        ng = 1
    x = np.empty((cells, species))
    it = np.zeros(ng, np.int64)
    rep = RefReport()
    st = ref().ref_solve_batch(strategy, k, species, cells, ptr(np.ascontiguousarray(row_ptr, np.int32)),
                               ptr(np.ascontiguousarray(col_idx, np.int32)), ptr(np.ascontiguousarray(values)),
                               ptr(np.ascontiguousarray(rhs)), tol, max_iter, mtpb, workers, ptr(x), ptr(it),
                               C.byref(rep))
    return st, BatchResult(x, it, None, None, rep)


def csr64(row_ptr, col_idx):
    return np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int64)


def orc_solve_single(algo, row_ptr, col_idx, vals, b, x0, tol, max_iter, ranges=None):
    n = len(row_ptr) - 1
    rp, ci = csr64(row_ptr, col_idx)
    ranges = np.array([[0, n]] if ranges is None else ranges, np.int64).reshape(-1)
    x = np.empty(n)
    out = OrcOutcome()
    fn = orc().orc_bicg_solve if algo == 0 else orc().orc_bicgstab_solve
    st = fn(n, ptr(rp), ptr(ci), ptr(np.ascontiguousarray(vals, np.float64)), ptr(np.ascontiguousarray(b, np.float64)),
            ptr(np.ascontiguousarray(x0 if x0 is not None else np.zeros(n), np.float64)), tol, max_iter, ptr(ranges),
            len(ranges) // 2, ptr(x), C.byref(out))
    return st, x, out


def ref_bicg_single(row_ptr, col_idx, vals, b, x0, tol, max_iter, ranges=None, host_stage=False):
    n = len(row_ptr) - 1
    rp, ci = csr64(row_ptr, col_idx)
    ranges = np.array([[0, n]] if ranges is None else ranges, np.int64).reshape(-1)
    x = np.empty(n)
    it, rms, cv, bd = _i64(), _f64(), _i32(), _i32()
    st = ref().ref_bicg_solve(n, ptr(rp), ptr(ci), ptr(np.ascontiguousarray(vals, np.float64)),
                              ptr(np.ascontiguousarray(b, np.float64)),
                              ptr(np.ascontiguousarray(x0 if x0 is not None else np.zeros(n), np.float64)), tol,
                              max_iter, ptr(ranges), len(ranges) // 2, int(host_stage), ptr(x), C.byref(it),
                              C.byref(rms), C.byref(cv), C.byref(bd))
    return st, x, OrcOutcome(it.value, rms.value, cv.value, bd.value)


def lu_solve(which, row_ptr, col_idx, vals, b):
    n = len(row_ptr) - 1
    rp, ci = csr64(row_ptr, col_idx)
    x = np.empty(n)
    lib = orc() if which == "orc" else ref()
    fn = lib.orc_lu_solve_csr if which == "orc" else lib.ref_lu_solve
    st = fn(n, ptr(rp), ptr(ci), ptr(np.ascontiguousarray(vals, np.float64)), ptr(np.ascontiguousarray(b, np.float64)),
            ptr(x))
    return st, x


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.float64).view(np.uint64)
