"""One Block-cells solve for ncu: python tools/prof_block.py [cells] [algo] [regime]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_17363_b200 import (REGIME_C, REGIME_P, Algo, BatchedSystem, DeviceSpec, Mechanism,  # noqa: E402
                                   Solver)

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
algo = Algo.BICG if (len(sys.argv) > 2 and sys.argv[2] == "bicg") else Algo.BICGSTAB_JACOBI
reg = REGIME_C if (len(sys.argv) > 3 and sys.argv[3] == "C") else REGIME_P
species = int(os.environ.get("SPECIES", "156"))
m = Mechanism(species, 3 * species, 0)
v, b = m.newton_batch(0, cells, cells, reg.h)
s = Solver(0)
sysm = BatchedSystem(species, cells, m.row_ptr, m.col_idx, torch.from_numpy(v).cuda(), torch.from_numpy(b).cuda())
for _ in range(int(os.environ.get("REPS", "1"))):
    kk = os.environ.get("K", "1")
    rep = s.solve_block_cells(sysm, None if kk == "N" else int(kk), DeviceSpec(), reg.tol, reg.max_iter, algo=algo,
                              timing=True)
    print(f"cells={cells} algo={algo.name} regime={reg.name} it_sum={rep.iterations_sum} "
          f"device_ms={rep.device_ms:.3f} -> {cells / rep.device_ms * 1e3:.0f} cell-solves/s", flush=True)
