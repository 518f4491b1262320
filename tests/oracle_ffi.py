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
        lib.ref_bicgstab_solve.argtypes = lib.ref_bicg_solve.argtypes
        lib.ref_batch_create.restype = _p
        lib.ref_batch_create.argtypes = [_i64, _i64, _p, _p, _p, _p]
        lib.ref_batch_destroy.argtypes = [_p]
        lib.ref_batch_run.argtypes = [_p, C.c_int, C.c_int, _i64, _f64, _i64, _i64, _i64, _p, _p, _p, _p,
                                      C.POINTER(RefReport)]
        lib.ref_solve_batch_bicgstab.argtypes = [C.c_int, _i64, _i64, _i64, _p, _p, _p, _p, _f64, _i64, _i64, _i64,
                                                 _p, _p, _p, _p, C.POINTER(RefReport)]
        lib.ref_tree_reduce.restype = _f64
        lib.ref_tree_reduce.argtypes = [_p, _i64, _i64]
        lib.ref_plan_reduce.restype = _f64
        lib.ref_plan_reduce.argtypes = [_p, _i64, _p, _i64]
        lib.ref_mechanism_pattern.argtypes = [_i64, _i64, C.c_uint64, C.POINTER(_i64), _p, _p]
        lib.ref_newton_batch.argtypes = [_i64, _i64, C.c_uint64, _i64, _i64, _i64, C.c_int, _f64, _p, _p]
        lib.ref_format_double.argtypes = [_f64, C.c_char_p]
        lib.ref_to_csv.argtypes = [_i64, _p, C.c_char_p] + [_p] * 9
        lib.ref_summary_roundtrip.argtypes = [C.c_char_p, _i64, _i64, _i64, _f64, C.c_int, _i64, _p, _p, _f64, _i64,
                                              C.c_uint64, _i64, C.c_char_p]
        lib.ref_plan_json.argtypes = [C.c_int, _i64, _i64, _i64, _i64]
        lib.ref_last_text.restype = C.c_char_p
        lib.ref_run_simulation.argtypes = [_i64, _i64, C.c_uint64, _i64, C.c_int, _i64, _f64, _f64, _i64, C.c_int,
                                           _i64, C.c_int, _f64, _i64, _i64, _p, _p, C.POINTER(_i64)]
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


def ref_solve_batch_bicgstab(strategy, k, row_ptr, col_idx, values, rhs, tol, max_iter, mtpb=1024, workers=1,
                             x=None):
    """Jacobi-BiCGSTAB through the reference's own primitives and drivers
    (oracle/ref_bicgstab.cpp): the checker of the north-star path.  Same
    outputs as orc_solve_batch (x, per-group iterations / rms / flags)."""
    species = len(row_ptr) - 1
    cells = values.shape[0]
    ng = orc().orc_group_count(strategy, cells, species, mtpb, k)
    if ng < 0:
        ng = 1
    x = np.empty((cells, species)) if x is None else x
    it = np.zeros(ng, np.int64)
    rms = np.zeros(ng)
    fl = np.zeros(ng, np.uint8)
    rep = RefReport()
    st = ref().ref_solve_batch_bicgstab(strategy, k, species, cells, ptr(np.ascontiguousarray(row_ptr, np.int32)),
                                        ptr(np.ascontiguousarray(col_idx, np.int32)), ptr(np.ascontiguousarray(values)),
                                        ptr(np.ascontiguousarray(rhs)), tol, max_iter, mtpb, workers, ptr(x), ptr(it),
                                        ptr(rms), ptr(fl), C.byref(rep))
    return st, BatchResult(x, it, rms, fl, rep)


class RefBatch:
    """The reference's host BatchedSystem (strategies.hpp:15-23), built once
    in oracle/_ref and solved repeatedly: run(algo=0) is the stock
    run_strategy (BiCG), run(algo=1) the composed Jacobi-BiCGSTAB."""

    def __init__(self, row_ptr, col_idx, values, rhs):
        self.species = len(row_ptr) - 1
        self.cells = values.shape[0]
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        self.h = ref().ref_batch_create(self.species, self.cells, ptr(self.row_ptr),
                                        ptr(np.ascontiguousarray(col_idx, np.int32)),
                                        ptr(np.ascontiguousarray(values)), ptr(np.ascontiguousarray(rhs)))
        if not self.h:
            raise MemoryError("ref_batch_create failed")

    def run(self, algo, strategy, k, tol, max_iter, mtpb=1024, workers=1, x=None):
        ng = orc().orc_group_count(strategy, self.cells, self.species, mtpb, k)
        ng = max(ng, 1)
        x = np.empty((self.cells, self.species)) if x is None else x
        it = np.zeros(ng, np.int64)
        rms = np.zeros(ng) if algo == 1 else None
        fl = np.zeros(ng, np.uint8) if algo == 1 else None
        rep = RefReport()
        st = ref().ref_batch_run(self.h, algo, strategy, k, tol, max_iter, mtpb, workers, ptr(x), ptr(it), ptr(rms),
                                 ptr(fl), C.byref(rep))
        return st, BatchResult(x, it, rms, fl, rep)

    def close(self):
        if self.h:
            ref().ref_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def ref_solve_checker(algo, strategy, k, row_ptr, col_idx, values, rhs, tol, max_iter, mtpb=1024, workers=1):
    """The strongest checker available for `algo` (0 BiCG, 1 Jacobi-BiCGSTAB):
    the compiled reference (BiCG: run_strategy; BiCGSTAB: its primitives
    composed) when oracle/_ref exists, else the C restatement.  Returns
    (status, BatchResult with x/iters/rms/flags, kind)."""
    if have_ref():
        if algo == 1:
            st, r = ref_solve_batch_bicgstab(strategy, k, row_ptr, col_idx, values, rhs, tol, max_iter, mtpb,
                                             workers)
            return st, r, "reference primitives (oracle/_ref ref_solve_batch_bicgstab)"
    st, r = orc_solve_batch(strategy, algo, k, row_ptr, col_idx, values, rhs, tol, max_iter, mtpb, workers)
    return st, r, "C restatement (oracle/liborc)"


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


def ref_bicgstab_single(row_ptr, col_idx, vals, b, x0, tol, max_iter, ranges=None, host_stage=False):
    n = len(row_ptr) - 1
    rp, ci = csr64(row_ptr, col_idx)
    ranges = np.array([[0, n]] if ranges is None else ranges, np.int64).reshape(-1)
    x = np.empty(n)
    it, rms, cv, bd = _i64(), _f64(), _i32(), _i32()
    st = ref().ref_bicgstab_solve(n, ptr(rp), ptr(ci), ptr(np.ascontiguousarray(vals, np.float64)),
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


# --- run_simulation (simulate.cpp:72-178) ------------------------------------

STEP_FIELDS = ("step", "newton_iterations", "iterations_effective", "iterations_sum", "max_residual_rms",
               "wall_time_ns", "breakdown_fallbacks", "clip_events")


class RefStepStats(C.Structure):
    _fields_ = [(f, _f64 if f == "max_residual_rms" else _i64) for f in STEP_FIELDS]


class SimOut:
    def __init__(self, states, per_step, abort_step):
        self.states, self.per_step, self.abort_step = states, per_step, abort_step


def ref_run_simulation(species, reactions, seed, cells, mode, steps, dt, tol, max_iter, strategy, k, direct,
                       newton_rtol=1e-10, max_newton=10, states=None, workers=1):
    """The reference's own run_simulation (oracle/_ref).  strategy: 0 one-cell,
    1 multi-cells, 2 block-cells (k 0 = "N")."""
    y = np.ones((cells, species)) if states is None else np.array(states, np.float64, order="C", copy=True)
    stats = (RefStepStats * max(1, steps))()
    ab = _i64(-1)
    st = ref().ref_run_simulation(species, reactions, seed, cells, mode, steps, dt, tol, max_iter, strategy, k,
                                  int(direct), newton_rtol, max_newton, workers, ptr(y), stats, C.byref(ab))
    per_step = [{f: getattr(stats[i], f) for f in STEP_FIELDS} for i in range(steps)] if st == 0 else []
    return st, SimOut(y, per_step, ab.value)


def orc_run_simulation(mech, cells, mode, steps, dt, tol, max_iter, strategy, k, algo, direct, newton_rtol=1e-10,
                       max_newton=10, states=None, workers=8):
    """Restatement of run_simulation (simulate.cpp:72-178) over the checkers:
    the workload generator's Newton systems (bcw_newton_batch: A = I - hJ(y),
    b = -(y - y_prev - h f(y)), simulate.cpp:29-42) solved by the C oracle
    (orc_solve_batch, any algorithm) or its dense LU (direct), then the
    update, the max-norm Newton test, SolverAbort on a non-finite state and
    end-of-step clipping, in the reference's order.  Returns (status, SimOut):
    status -9 = SolverAbort (abort_step set)."""
    y = np.ones((cells, mech.species)) if states is None else np.array(states, np.float64, order="C", copy=True)
    per_step = []
    for step in range(steps):
        prev = y.copy()
        rec = dict(step=step, newton_iterations=0, iterations_effective=0, iterations_sum=0, max_residual_rms=0.0,
                   wall_time_ns=0, breakdown_fallbacks=0, clip_events=0)
        for newton in range(1, max_newton + 1):
            v, b = mech.newton_batch(0, cells, cells, dt, mode, y=y, y_prev=prev)
            if direct:
                dx = np.empty_like(y)
                for c in range(cells):
                    st, dx[c] = lu_solve("orc", mech.row_ptr, mech.col_idx, v[c], b[c])
                    if st != 0:
                        return st, SimOut(y, per_step, -1)
            else:
                st, res = orc_solve_batch(strategy, algo, k, mech.row_ptr, mech.col_idx, v, b, tol, max_iter,
                                          workers=workers)
                if st != 0:
                    return st, SimOut(y, per_step, -1)
                dx = res.x
                rec["iterations_effective"] += res.report.iterations_effective
                rec["iterations_sum"] += res.report.iterations_sum
                rec["max_residual_rms"] = max(rec["max_residual_rms"], res.report.max_residual_rms)
                rec["breakdown_fallbacks"] += res.report.breakdown_fallbacks
            update_inf = float(np.fmax.reduce(np.abs(dx).ravel(), initial=0.0))  # std::max keeps a on NaN
            y = y + dx
            rec["newton_iterations"] = newton
            if not np.isfinite(y).all():
                return -9, SimOut(y, per_step, step)
            state_inf = float(np.abs(y).max(initial=0.0))
            if update_inf < newton_rtol * state_inf:
                break
        neg = y < 0.0
        rec["clip_events"] = int(neg.sum())
        y[neg] = 0.0
        per_step.append(rec)
    return 0, SimOut(y, per_step, -1)
