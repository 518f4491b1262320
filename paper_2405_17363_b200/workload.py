"""Synthetic CB05-shaped workloads (include/blockcells_workload.h).

``Mechanism(156, 468, 0)`` is the reference's M156 (nnz 1556) and
``Mechanism(312, 936, 0)`` its M312 (nnz 3032).
``newton_batch`` returns the first backward-Euler Newton system of step 0 for
a range of cells, bit-identical to the reference's
``newton_system(M, cell_conditions(c, C, mode), y=1, y_prev=1, h)``.
Regimes: P (paper) h=120 s, tol=1e-30, max_iter=1000; C (converging) h=1 s,
tol=1e-10.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import _native

IDEAL, REALISTIC = 0, 1


@dataclass(frozen=True)
class Regime:
    name: str
    h: float
    tol: float
    max_iter: int


REGIME_P = Regime("P", 120.0, 1e-30, 1000)
REGIME_C = Regime("C", 1.0, 1e-10, 1000)


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


class Mechanism:
    def __init__(self, species: int = 156, reactions: Optional[int] = None, seed: int = 0):
        self.lib = _native.workload()
        reactions = 3 * species if reactions is None else reactions
        self._m = C.c_void_p()
        st = self.lib.bcw_mechanism_create(species, reactions, seed, C.byref(self._m))
        if st != 0:
            raise ValueError(f"generate_mechanism({species}, {reactions}, {seed}) failed: {st}")
        self.species, self.reactions, self.seed = species, reactions, seed
        self.nnz = int(self.lib.bcw_nnz(self._m))
        self.row_ptr = np.zeros(species + 1, np.int32)
        self.col_idx = np.zeros(self.nnz, np.int32)
        self.lib.bcw_pattern(self._m, _p(self.row_ptr), _p(self.col_idx))

    def __del__(self):
        try:
            if self._m:
                self.lib.bcw_mechanism_destroy(self._m)
                self._m = C.c_void_p()
        except Exception:
            pass

    def newton_batch(self, first: int, count: int, total_cells: int, h: float, mode: int = REALISTIC,
                     y: Optional[np.ndarray] = None, y_prev: Optional[np.ndarray] = None,
                     values: Optional[np.ndarray] = None, rhs: Optional[np.ndarray] = None,
                     threads: int = 0) -> Tuple[np.ndarray, np.ndarray]:
        values = np.empty((count, self.nnz), np.float64) if values is None else values
        rhs = np.empty((count, self.species), np.float64) if rhs is None else rhs
        for name, a, shape in (("values", values, (count, self.nnz)), ("rhs", rhs, (count, self.species)),
                               ("y", y, (count, self.species)), ("y_prev", y_prev, (count, self.species))):
            if a is None:
                continue
            if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.shape != shape or \
                    not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"newton_batch: {name} must be a C-contiguous float64 array of shape {shape}")
        st = self.lib.bcw_newton_batch(self._m, first, count, total_cells, mode, float(h), _p(y), _p(y_prev),
                                       _p(values), _p(rhs), threads)
        if st != 0:
            raise ValueError(f"bcw_newton_batch failed: {st}")
        return values, rhs

    def rate_constants(self, first: int, count: int, total_cells: int, mode: int = REALISTIC,
                       threads: int = 0) -> np.ndarray:
        rates = np.empty((count, self.reactions), np.float64)
        st = self.lib.bcw_rate_constants(self._m, first, count, total_cells, mode, _p(rates), threads)
        if st != 0:
            raise ValueError(f"bcw_rate_constants failed: {st}")
        return rates

    def stamp_program(self) -> dict:
        ns = int(self.lib.bcw_stamp_count(self._m))
        nr = self.reactions
        out = dict(stamp_ptr=np.zeros(nr + 1, np.int32), stamp_slot=np.zeros(max(ns, 1), np.int32),
                   stamp_sign=np.zeros(max(ns, 1), np.float64), stamp_other=np.zeros(max(ns, 1), np.int32),
                   reactant_ptr=np.zeros(nr + 1, np.int32), reactants=np.zeros(2 * nr + 1, np.int32),
                   product_ptr=np.zeros(nr + 1, np.int32), products=np.zeros(2 * nr + 1, np.int32),
                   diag_slot=np.zeros(self.species, np.int32))
        self.lib.bcw_stamp_program(self._m, *[_p(out[k]) for k in (
            "stamp_ptr", "stamp_slot", "stamp_sign", "stamp_other", "reactant_ptr", "reactants",
            "product_ptr", "products", "diag_slot")])
        return out


def assemble_on_device(solver, mech: Mechanism, first: int, count: int, total_cells: int, h: float,
                       mode: int = REALISTIC, stream=None):
    """Newton systems assembled by the CUDA kernel (bc_newton_assemble) into
    CUDA tensors (values (count, nnz), rhs (count, species))."""
    import torch
    lib = _native.b200()
    dev = torch.device("cuda", solver.device)
    prog = {k: torch.from_numpy(v).to(dev) for k, v in mech.stamp_program().items()}
    rates = torch.from_numpy(mech.rate_constants(first, count, total_cells, mode)).to(dev)
    values = torch.empty((count, mech.nnz), dtype=torch.float64, device=dev)
    rhs = torch.empty((count, mech.species), dtype=torch.float64, device=dev)
    vp = lambda t: C.c_void_p(t.data_ptr())
    st = lib.bc_newton_assemble(solver._ctx, count, mech.species, mech.reactions, mech.nnz, vp(rates),
                                *[vp(prog[k]) for k in ("stamp_ptr", "stamp_slot", "stamp_sign", "stamp_other",
                                                         "reactant_ptr", "reactants", "product_ptr", "products",
                                                         "diag_slot")],
                                float(h), None, None, vp(values), vp(rhs),
                                C.c_void_p(stream) if stream else None)
    if st != 0:
        raise RuntimeError(lib.bc_last_error(solver._ctx).decode())
    return values, rhs
