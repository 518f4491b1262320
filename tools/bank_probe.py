"""Run under ncu to measure LDS.64 wavefronts for named slot patterns:
  ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum \
      -k regex:bank_probe python tools/bank_probe.py
Each launch = one pattern (order printed), T steps x iters loads per warp."""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
lib = C.CDLL(os.path.join(HERE, "libmicrobench.so"))
lib.mb_bank_probe.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
pats = {}
L = np.arange(32)
pats["identity"] = [L]
pats["same_pair_all32"] = [L * 16]
pats["half0_pair0_half1_pair1"] = [np.where(L < 16, L * 16, (L - 16) * 16 + 1)]
pats["quarter_pairs"] = [np.where(L < 8, L * 16, np.where(L < 16, (L - 8) * 16 + 1, L))]
pats["two_per_pair_spread"] = [(L % 16) + 16 * (L // 16)]  # each pair 2 distinct, one per half
pats["two_per_pair_samehalf"] = [np.where(L < 16, (L // 2) + 16 * (L % 2), L)]  # half0: pairs 0-7 x2
pats["broadcast"] = [np.zeros(32, int)]
pats["lanes_pair_by_lane_mod8"] = [(L % 8) + 16 * (L // 8)]  # 4 distinct in each of 8 pairs
pats["rand156"] = [np.random.default_rng(0).integers(0, 156, 32) for _ in range(8)]
# the real M156 schedules (identity placement vs annealed placement)
try:
    from test_capi import export_schedule
    from paper_2405_17363_b200 import Mechanism
    m = Mechanism(156, 468, 0)
    sc = export_schedule(m.row_ptr, m.col_idx, 1, 0)
    w = sc["words"].reshape(sc["S"], 32) & 0xFFF
    pats["m156_sched_current"] = [w[t] for t in range(min(sc["S"], 64))]
except Exception as e:  # noqa
    print("no schedule:", e)
ms = C.c_double()
for name, rows in pats.items():
    tab = np.ascontiguousarray(np.array(rows, np.uint32).reshape(-1))
    T = len(rows)
    assert lib.mb_bank_probe(C.c_void_p(tab.ctypes.data), T, 200, 4, C.byref(ms)) == 0
    print(f"pattern {name}: T={T} loads_per_warp={T * 200}", flush=True)
