"""BASELINE.json config 3 (and 5): Block-cells(1) vs Block-cells(N) vs
Multi-cells vs one-thread-per-cell on 100k CB05-sized cells, both regimes,
device-resident, CUDA-event timed.  Writes gpurun_out/strategies.json.
    python tools/compare_strategies.py [cells] [species]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_17363_b200 import (REGIME_C, REGIME_P, Algo, BatchedSystem, DeviceSpec, Mechanism,  # noqa: E402
                                   Solver, Strategy, StrategyConfig)

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
species = int(sys.argv[2]) if len(sys.argv) > 2 else 156
m = Mechanism(species, 3 * species, 0)
s = Solver(0)
out = []
for reg in (REGIME_P, REGIME_C):
    v, b = m.newton_batch(0, cells, cells, reg.h)
    sysm = BatchedSystem(species, cells, m.row_ptr, m.col_idx, torch.from_numpy(v).cuda(), torch.from_numpy(b).cuda())
    for algo in (Algo.BICGSTAB_JACOBI, Algo.BICG):
        for name, cfg in (("block-cells(1)", StrategyConfig(Strategy.BlockCells, 1)),
                          ("block-cells(N)", StrategyConfig(Strategy.BlockCells, None)),
                          ("multi-cells", StrategyConfig(Strategy.MultiCells)),
                          ("thread-per-cell", StrategyConfig(Strategy.ThreadPerCell))):
            n = cells  # every strategy on the whole batch (BASELINE.json configs[2])
            sub = BatchedSystem(species, n, m.row_ptr, m.col_idx, sysm.values[:n], sysm.rhs[:n])
            best = None
            for _ in range(1 if name == "thread-per-cell" and reg.name == "P" else 2):  # ~10-20 s each
                rep = s.run_strategy(sub, cfg, DeviceSpec(), reg.tol, reg.max_iter, 1, algo, timing=True)
                best = rep if best is None or rep.device_ms < best.device_ms else best
            row = dict(regime=reg.name, algo=algo.name, strategy=name, cells=n, device_ms=best.device_ms,
                       cell_solves_per_s=n / best.device_ms * 1e3, iterations_effective=best.iterations_effective,
                       iterations_sum=best.iterations_sum, fallbacks=best.breakdown_fallbacks)
            print(json.dumps(row), flush=True)
            out.append(row)
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/strategies_m{species}.json", "w") as f:
    json.dump(out, f, indent=1)
