"""Small-batch sweep: cell-solves/s of M156 P-regime Block-cells(1) solves vs
batch size, latency kernel (BC_LATENCY=1) against the throughput kernel
(BC_LATENCY=0), kernel time by CUDA events (best of REPS), SM clock sampled.
Run under gpurun: python tools/latency_sweep.py [algo] > out.jsonl"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_17363_b200 import REGIME_P, Algo, BatchedSystem, DeviceSpec, Mechanism, Solver  # noqa: E402

algo = Algo.BICG if (len(sys.argv) > 1 and sys.argv[1] == "bicg") else Algo.BICGSTAB_JACOBI
species = int(os.environ.get("SPECIES", "156"))
m = Mechanism(species, 3 * species, 0)
s = Solver(0)
for cells in [int(c) for c in os.environ.get("CELLS", "1,10,50,100,148,200,296,444,592,1184,2368,10000").split(",")]:
    v, b = m.newton_batch(0, cells, cells, REGIME_P.h)
    sysm = BatchedSystem(species, cells, m.row_ptr, m.col_idx, torch.from_numpy(v).cuda(), torch.from_numpy(b).cuda())
    for mode in ("1", "0"):
        os.environ["BC_LATENCY"] = mode
        s.solve_block_cells(sysm, 1, DeviceSpec(), REGIME_P.tol, REGIME_P.max_iter, algo=algo)
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "100"],
                               stdout=subprocess.PIPE, text=True)
        best = None
        for _ in range(int(os.environ.get("REPS", "5"))):
            rep = s.solve_block_cells(sysm, 1, DeviceSpec(), REGIME_P.tol, REGIME_P.max_iter, algo=algo, timing=True)
            best = rep.device_ms if best is None else min(best, rep.device_ms)
        smi.terminate()
        clk = [float(x) for x in smi.communicate()[0].split() if x.replace(".", "").isdigit()]
        print(json.dumps({"cells": cells, "latency_mode": mode == "1", "algo": algo.name, "species": species,
                          "kernels": rep.kernels, "device_ms": best, "cell_solves_per_s": cells / best * 1e3,
                          "sm_mhz": sorted(clk)[len(clk) // 2] if clk else None,
                          "iterations_sum": rep.iterations_sum}), flush=True)
