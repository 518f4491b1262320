"""Measure the B200 ceilings that bound the fused solver (FP64 issue rate,
shared-memory gather rate, warp shuffles).  Writes profiles/microbench_b200.json.
    python tools/microbench.py"""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmicrobench.so")
if not os.path.exists(LIB):
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false",
                    "-shared", "-Xcompiler", "-fPIC", "-o", LIB, os.path.join(HERE, "microbench.cu")], check=True)
lib = C.CDLL(LIB)
lib.mb_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_double)]
sms = 148
out = {}
ms = C.c_double()
for name, which in (("dadd", 0), ("dmul", 1), ("dfma", 2)):
    blocks, threads, iters = sms * 8, 256, 4096
    assert lib.mb_run(which, blocks, threads, iters, None, C.byref(ms)) == 0
    ops = blocks * threads * iters * 8
    out[f"{name}_Gops"] = ops / (ms.value / 1e3) / 1e9
    out[f"{name}_per_clk_per_sm_at_1965MHz"] = ops / (ms.value / 1e3) / 1.965e9 / sms
rng = np.random.default_rng(0)
idx = rng.integers(0, 156, 64 * 32).astype(np.uint32)
for name, which in (("lds64_seq", 3), ("lds64_random156", 4)):
    blocks, iters = sms * 8, 2048
    assert lib.mb_run(which, blocks, 256, iters, C.c_void_p(idx.ctypes.data), C.byref(ms)) == 0
    loads = blocks * 256 * iters * 64
    out[f"{name}_Gloads"] = loads / (ms.value / 1e3) / 1e9
    out[f"{name}_lanes_per_clk_per_sm"] = loads / (ms.value / 1e3) / 1.965e9 / sms
assert lib.mb_run(5, sms * 8, 256, 4096, None, C.byref(ms)) == 0
sh = sms * 8 * 256 * 4096 * 5
out["shfl64_butterfly_steps_G_per_s"] = sh / (ms.value / 1e3) / 1e9
out["shfl64_lane_steps_per_clk_per_sm"] = sh / (ms.value / 1e3) / 1.965e9 / sms
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "microbench_b200.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))

# TMEM reads (tcgen05.ld 32x32b.x16) alone / with random LDS.64 gathers / gathers alone
lib.mb_tmem.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_double)]
tm = {}
for warps in (4, 8, 16):
    for mode, name in ((0, "tmem"), (1, "tmem+lds"), (2, "lds")):
        iters = 2000
        st = lib.mb_tmem(mode, warps, iters, C.c_void_p(idx.ctypes.data), C.byref(ms))
        assert st == 0, st
        cyc = ms.value / 1e3 * 1.965e9
        tm[f"{name}_w{warps}_ms"] = ms.value
        if mode != 2:
            tm[f"{name}_w{warps}_tmem_B_per_clk_per_sm"] = warps * iters * 4 * 2 * 2048 / cyc
        if mode != 0:
            tm[f"{name}_w{warps}_lds_lanes_per_clk_per_sm"] = warps * iters * 4 * 8 * 32 / cyc
out["tmem"] = tm
with open(os.path.join(ROOT, "gpurun_out", "microbench_b200.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(tm, indent=1))
