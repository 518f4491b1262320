"""Where the end-to-end step goes: python tools/e2e_probe.py [cells]
Prints per-step wall time of run_strategy, of the bc_solve call inside it,
the pinned H2D bandwidth, and the device-resident step for comparison."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_17363_b200 import (REGIME_P, Algo, BatchedSystem, DeviceSpec, Mechanism, Solver, Strategy,  # noqa: E402
                                   StrategyConfig)

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
m = Mechanism(156, 468, 0)
v = torch.empty((cells, m.nnz), dtype=torch.float64, pin_memory=True).numpy()
b = torch.empty((cells, m.species), dtype=torch.float64, pin_memory=True).numpy()
m.newton_batch(0, cells, cells, REGIME_P.h, values=v, rhs=b)
x = torch.empty((cells, m.species), dtype=torch.float64, pin_memory=True).numpy()
s = Solver(0)
cfg = StrategyConfig(Strategy.BlockCells, 1)
hsys = BatchedSystem(m.species, cells, m.row_ptr, m.col_idx, v, b)
dv = torch.from_numpy(v).cuda()
t0 = time.perf_counter()
for _ in range(5):
    dv.copy_(torch.from_numpy(v), non_blocking=True)
torch.cuda.synchronize()
print(f"H2D pinned: {5 * v.nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
for i in range(4):
    t0 = time.perf_counter()
    rep = s.run_strategy(hsys, cfg, DeviceSpec(), REGIME_P.tol, REGIME_P.max_iter, 1, Algo.BICGSTAB_JACOBI, x_out=x,
                         timing=True)
    t1 = time.perf_counter()
    print(f"host step {1e3 * (t1 - t0):.1f} ms, bc_solve {rep.wall_time_ns / 1e6:.1f} ms, "
          f"device_ms {rep.device_ms:.1f}, launches {rep.kernel_launches}")
