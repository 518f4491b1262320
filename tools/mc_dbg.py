import sys, time, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from fixtures import random_batch
from paper_2405_17363_b200 import *
s = Solver(0)
rng = np.random.default_rng(7)
rp, ci, v, b = random_batch(rng, 4, 13)
sysm = BatchedSystem(13, 4, rp, ci, v, b)
t=time.time(); rep = s.run_strategy(sysm, StrategyConfig(Strategy.MultiCells), DeviceSpec(), 1e-12, 50, 1, Algo.BICG); print('small multi', rep.iterations_effective, time.time()-t, flush=True)
rp, ci, v, b = random_batch(rng, 90, 13)
sysm = BatchedSystem(13, 90, rp, ci, v, b)
t=time.time(); rep = s.run_strategy(sysm, StrategyConfig(Strategy.MultiCells), DeviceSpec(), 1e-12, 500, 1, Algo.BICG); print('90-cell multi', rep.iterations_effective, time.time()-t, flush=True)
m = Mechanism(156,468,0); v,b = m.newton_batch(0,100,100,120.0)
sysm = BatchedSystem(156, 100, m.row_ptr, m.col_idx, v, b)
t=time.time(); rep = s.run_strategy(sysm, StrategyConfig(Strategy.MultiCells), DeviceSpec(), 1e-30, 1000, 1, Algo.BICG); print('m156 multi P', rep.iterations_effective, time.time()-t, flush=True)
