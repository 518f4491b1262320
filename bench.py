#!/usr/bin/env python
"""Benchmark: BiCGSTAB cell-solves/sec at 100k cells per B200 (BASELINE.json).

Workload (BASELINE.json configs[2]/[3]): mechanism M156
(generate_mechanism(156, 468, 0): 156 species, 1556 nnz), the first Newton
system of step 0 for every cell (A = I - hJ(1), b = h f(1), realistic
conditions over the GLOBAL cell index), P regime (h = 120 s, tol = 1e-30,
max_iter = 1000: every cell runs the full 1000 iterations), Block-cells(1),
Jacobi-preconditioned BiCGSTAB, fp64.  One step = one solve of the rank's
100k cells.  Multi-GPU: weak scaling, contiguous cell ranges per rank, no
collective on the data path (barrier + max-of-times only).

  value     device-resident: inputs already in HBM, CUDA events on the solve
            stream, max over ranks, cells of all ranks / time
  e2e       through the public API (Solver.run_strategy) with pinned HOST
            inputs: H2D of values+rhs, solve, D2H of x + per-group outputs
  roofline  dominant kernel (block_cells_tmem_kernel): algorithmic streaming
            bytes (it*(16*nnz+80*n)+16*n+16 per cell) / its event
            time, against MEASURED_PEAKS.json hbm_gbs (the metric's label); the
            binding resource (shared-memory pipe) from the planner's bank model,
            measured in this run, next to the committed ncu capture
  parity    the last timed step's output (every cell at N=1) against the
            checker -- Jacobi-BiCGSTAB composed from the reference's own
            compiled primitives (oracle/_ref), BiCG: the reference's
            run_strategy -- bit for bit: x, per-group iterations, rms, flags
  cpu_baseline  the same checker run is the reference's CPU path on all host
            threads over the whole workload (rank 0, N=1), plus bounded
            single-thread samples and the stock BiCG run_strategy
  bicg_companion  the reference's own algorithm (BiCG) on the GPU, same
            cells, for a like-for-like ratio against the stock reference

  --impl reference   times the reference's CPU implementation only: the
            whole workload every step through oracle/_ref (BiCGSTAB: composed
            from the reference's primitives and strategy drivers; BiCG: its
            stock run_strategy), inputs from the reference's own generator.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BiCGSTAB cell-solves/sec at 100k cells (1/2/4/8 B200); % HBM roofline"
UNIT = "cell-solves/s"
SPECIES, REACTIONS, SEED = 156, 468, 0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cells", type=int, default=100_000, help="cells per GPU")
    ap.add_argument("--species", type=int, default=SPECIES,
                    help="mechanism size: 156 (CB05-sized M156) or 312 (scaled M312, BASELINE.json configs[4])")
    ap.add_argument("--regime", default="P", choices=["P", "C"])
    ap.add_argument("--algo", default="bicgstab", choices=["bicgstab", "bicg"])
    ap.add_argument("--strategy", default="block-cells-1")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the bit-for-bit check of the last step")
    ap.add_argument("--parity-cells", type=int, default=100_000,
                    help="cells checked per run (all of them at N=1 up to this many; strided groups beyond)")
    ap.add_argument("--no-companion", action="store_true", help="skip the GPU BiCG companion measurement")
    ap.add_argument("--no-dropin", action="store_true",
                    help="skip e2e_dropin (blockcells::run_strategy through the C++ drop-in, tests/cpp/bin/dropin_bench)")
    return ap.parse_args()


def regime(name):
    from paper_2405_17363_b200 import REGIME_C, REGIME_P
    return REGIME_P if name == "P" else REGIME_C


def algorithmic_bytes(iters, n, nnz):
    """B_cell = it*(16*nnz + 80*n) + 16*n + 16."""
    return float(sum(int(i) * (16 * nnz + 80 * n) + 16 * n + 16 for i in iters))


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of block_cells_kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_block_cells_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_reference_rate(values, rhs, row_ptr, col_idx, reg, budget_s, algo_name="bicg", threads=None,
                       cfg_code=(2, 1)):
    """The reference's CPU path (oracle/_ref: BiCG = its stock run_strategy,
    BiCGSTAB = composed from its primitives; the C restatement only where
    oracle/_ref is absent) on a bounded prefix sample of the workload, all host
    threads unless `threads`.  Returns (rate, cores, sample, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as of
    cores = threads or os.cpu_count() or 1
    algo = 0 if algo_name == "bicg" else 1
    strat, k = cfg_code
    use_ref = of.have_ref()
    kind = "reference" if use_ref else "port"

    def run(nc):
        """Seconds of solver time: SolveReport::wall_time_ns (the whole
        run_strategy call, strategies.cpp:241-247) for oracle/_ref, wall clock
        for the port."""
        if use_ref:
            rb = of.RefBatch(row_ptr, col_idx, values[:nc], rhs[:nc])
            st, res = rb.run(algo, strat, k, reg.tol, reg.max_iter, workers=cores)
            rb.close()
            assert st == 0, st
            return res.report.wall_time_ns / 1e9
        t0 = time.perf_counter()
        st, res = of.orc_solve_batch(strat, algo, k, row_ptr, col_idx, values[:nc], rhs[:nc], reg.tol, reg.max_iter,
                                     workers=cores)
        assert st == 0, st
        return time.perf_counter() - t0

    probe = min(len(values), 4 * cores)
    dt = run(probe)
    nc = int(min(len(values), max(probe, probe * budget_s / max(dt, 1e-3))))
    dt = run(nc)
    solver = (("reference run_strategy (BiCG)" if algo == 0 else
               "Jacobi-BiCGSTAB composed from the reference's primitives") if use_ref
              else f"C restatement {algo_name}")
    sample = f"{solver}, first {nc} cells of the workload, {cores} threads, {dt:.1f} s"
    return nc / dt, cores, sample, kind


def strategy_config(name):
    """block-cells-1 (default) / block-cells-<k> / block-cells-N / one-cell / multi-cells / thread-per-cell"""
    from paper_2405_17363_b200 import Strategy, StrategyConfig
    if name.startswith("block-cells-"):
        k = name.rsplit("-", 1)[-1]
        return StrategyConfig(Strategy.BlockCells, None if k == "N" else int(k))
    return {"one-cell": StrategyConfig(Strategy.OneCell), "multi-cells": StrategyConfig(Strategy.MultiCells),
            "thread-per-cell": StrategyConfig(Strategy.ThreadPerCell)}[name]


def dominant_kernel(bits):
    """The solver kernel that carries the step, from SolveReport.kernels."""
    from paper_2405_17363_b200 import KERNEL_BLOCK, KERNEL_MULTI, KERNEL_THREAD, KERNEL_TMEM
    for bit, name in ((KERNEL_TMEM, "block_cells_tmem_kernel"), (KERNEL_BLOCK, "block_cells_kernel"),
                      (KERNEL_MULTI, "multi_cells_kernel"), (KERNEL_THREAD, "thread_per_cell_kernel")):
        if bits & bit:
            return name
    return "lu_fallback_kernel"


def make_workload(cells, first, total, reg, species=SPECIES):
    import numpy as np
    from paper_2405_17363_b200 import Mechanism
    m = Mechanism(species, 3 * species, SEED)  # generate_mechanism(s, 3s, 0), bench.hpp:18,25,32
    try:
        import torch
        values = torch.empty((cells, m.nnz), dtype=torch.float64, pin_memory=torch.cuda.is_available()).numpy()
        rhs = torch.empty((cells, m.species), dtype=torch.float64, pin_memory=torch.cuda.is_available()).numpy()
    except Exception:
        values = np.empty((cells, m.nnz))
        rhs = np.empty((cells, m.species))
    m.newton_batch(first, cells, total, reg.h, values=values, rhs=rhs)
    return m, values, rhs


def bench_config(args, n, nnz, cells, n_total, reg, world):
    """The `config` both arms print (identical for the same flags)."""
    algo_label = "Jacobi-BiCGSTAB" if args.algo == "bicgstab" else "BiCG"
    return {
        "workload": (f"M{n} ({n} species, {nnz} nnz) first Newton system of step 0, {cells} cells/GPU "
                     f"({n_total} total), {args.strategy}, {algo_label}, "
                     f"{reg.name} regime (h={reg.h:g} s, tol={reg.tol:g}, max_iter={reg.max_iter})"),
        "cells_per_gpu": cells, "global_cells": n_total, "strategy": args.strategy,
        "algorithm": args.algo, "regime": reg.name,
        "l2": f"inputs larger than L2 ({cells * nnz * 8 / 1e9:.3f} GB values per GPU vs 126 MB L2)",
        "parallelism": (f"replicas over {world} GPU(s) (Multi-cells is one global system)"
                        if args.strategy == "multi-cells" and world > 1
                        else f"cell-range sharding over {world} GPU(s), no collectives"),
    }


def ref_strategy(name):
    """(strategy code, k) for oracle/_ref: 0 one-cell, 1 multi-cells, 2 block-cells (k 0 = N)."""
    if name.startswith("block-cells-"):
        k = name.rsplit("-", 1)[-1]
        return 2, 0 if k == "N" else int(k)
    return {"one-cell": (0, 0), "multi-cells": (1, 0), "thread-per-cell": (0, 0)}[name]


def reference_inputs(species, first, count, total, h):
    """The reference's own generator (mechanism.cpp / simulate.cpp:46-64 via
    oracle/_ref ref_newton_batch), in host threads over cell ranges."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as of
    lib = of.ref()
    nnz = of._i64()
    assert lib.ref_mechanism_pattern(species, 3 * species, SEED, of.C.byref(nnz), None, None) == 0
    rp = np.zeros(species + 1, np.int32)
    ci = np.zeros(nnz.value, np.int32)
    assert lib.ref_mechanism_pattern(species, 3 * species, SEED, of.C.byref(nnz), of.ptr(rp), of.ptr(ci)) == 0
    values = np.empty((count, nnz.value))
    rhs = np.empty((count, species))
    nt = max(1, min(os.cpu_count() or 1, 32))
    bounds = [count * t // nt for t in range(nt + 1)]

    def part(t):
        a, b = bounds[t], bounds[t + 1]
        if b > a:
            st = lib.ref_newton_batch(species, 3 * species, SEED, first + a, b - a, total, 1, h,
                                      of.ptr(values[a:b]), of.ptr(rhs[a:b]))
            assert st == 0, st
    ths = [threading.Thread(target=part, args=(t,)) for t in range(nt)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return rp, ci, values, rhs


def main_reference(args):
    """The reference's CPU path on the box's host cores, the WHOLE workload
    every step (rank 0 alone under torchrun): BiCGSTAB composed from the
    reference's compiled spmv/axpby/plan_reduce_map/lu_solve and its strategy
    drivers (oracle/ref_bicgstab.cpp), or for --algo bicg its stock
    run_strategy.  The BatchedSystem is built once (the reference's host form),
    so a step is exactly one solve; its time is the reference's own
    SolveReport::wall_time_ns clock.  The stock BiCG run_strategy is timed once
    beside it, so both algorithms have a reference number."""
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as of
    if not of.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbcref.so not built"}), flush=True)
        return
    reg = regime(args.regime)
    n_total = args.cells * world
    cells = args.cells
    rp, ci, values, rhs = reference_inputs(args.species, 0, cells, n_total, reg.h)
    nnz = int(rp[-1])
    strat, k = ref_strategy(args.strategy)
    cores = os.cpu_count() or 1
    algo = 1 if args.algo == "bicgstab" else 0
    rb = of.RefBatch(rp, ci, values, rhs)
    x = np.empty((cells, args.species))
    times = []
    st, res = rb.run(algo, strat, k, reg.tol, reg.max_iter, workers=cores, x=x)  # warm-up 1: the whole workload
    assert st == 0, st
    # Every step is the whole workload unless that would take the run past
    # ~7 minutes; then each step is the same contiguous prefix sample, sized
    # to fit (ms_per_step is always the measured time of what a step solved).
    per_step = res.report.wall_time_ns / 1e9
    sample = cells
    if per_step * (args.warmup + args.steps) > 420.0:
        sample = max(1, int(cells * 420.0 / (per_step * (args.warmup + args.steps))))
        if strat == 2 and k > 1:
            sample = max(k, sample // k * k)
        rb.close()
        rb = of.RefBatch(rp, ci, np.ascontiguousarray(values[:sample]), np.ascontiguousarray(rhs[:sample]))
        x = np.empty((sample, args.species))
    for i in range(1, args.warmup + args.steps):
        st, res = rb.run(algo, strat, k, reg.tol, reg.max_iter, workers=cores, x=x)
        assert st == 0, st
        if i >= args.warmup:
            times.append(res.report.wall_time_ns / 1e9)
    if args.warmup == 0:
        times.insert(0, per_step)
    total_s = sum(times)
    value = sample * args.steps / total_s
    impl = ("Jacobi-BiCGSTAB composed from the reference's compiled spmv/axpby/plan_reduce_map/lu_solve and its "
            "strategy drivers (oracle/_ref ref_bicgstab.cpp)" if algo == 1 else "the reference's stock run_strategy")
    extra = None
    if algo == 1:  # the reference's own algorithm, stock code path, once on the same cells
        st, r0 = rb.run(0, strat, k, reg.tol, reg.max_iter, workers=cores, x=x)
        assert st == 0, st
        extra = {"value": cells / (r0.report.wall_time_ns / 1e9), "unit": UNIT, "cores": cores,
                 "sample": f"stock run_strategy (BiCG) on all {cells} cells, one run, {cores} threads"}
    rb.close()
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, args.species, nnz, cells, n_total, reg, world),
        "reference_impl": impl,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": (f"{impl}: " + (f"all {cells} cells" if sample == cells else
                                                           f"the first {sample} of {cells} cells") +
                                    f" every step, {cores} threads, SolveReport::wall_time_ns")},
        "reference_bicg": extra,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def parity_check(args, rep, m, h_values, h_rhs, reg, cfg_code, k, budget_cells, threads):
    """Bit-for-bit check of one GPU solve against the checker on strided whole
    groups (all of them when budget_cells >= cells).  Returns the parity dict
    and, when every cell was checked, the checker's all-core timing."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as of
    strat, kk = cfg_code
    cells = h_values.shape[0]
    x_gpu = rep.per_cell_x.cpu().numpy() if hasattr(rep.per_cell_x, "cpu") else np.asarray(rep.per_cell_x)
    it_gpu = np.asarray(rep.per_block_iterations)
    ng = len(it_gpu)
    ksz = 1 if strat in (0,) else (k if strat == 2 else cells)
    gsize = np.full(ng, ksz, np.int64)
    gsize[-1] = cells - ksz * (ng - 1)
    gfirst = np.concatenate([[0], np.cumsum(gsize)[:-1]])
    stride = max(1, int(np.ceil(cells / max(1, budget_cells))))
    groups = np.arange(0, ng, stride)
    if stride > 1 and groups[-1] != ng - 1 and gsize[-1] != ksz:
        groups = np.append(groups, ng - 1)  # the remainder group goes last, as in the whole batch
    sel = np.concatenate([np.arange(gfirst[g], gfirst[g] + gsize[g]) for g in groups])
    v = np.ascontiguousarray(h_values[sel])
    b = np.ascontiguousarray(h_rhs[sel])
    algo = 1 if args.algo == "bicgstab" else 0
    t0 = time.perf_counter()
    if of.have_ref():
        rb = of.RefBatch(m.row_ptr, m.col_idx, v, b)
        st, res = rb.run(algo, strat, kk, reg.tol, reg.max_iter, workers=threads)
        rb.close()
        checker = ("oracle/_ref: Jacobi-BiCGSTAB composed from the reference's primitives" if algo == 1
                   else "oracle/_ref: the reference's run_strategy")
        secs = res.report.wall_time_ns / 1e9
    else:
        st, res = of.orc_solve_batch(strat, algo, kk, m.row_ptr, m.col_idx, v, b, reg.tol, reg.max_iter,
                                     workers=threads)
        checker = "oracle/liborc: the C restatement"
        secs = time.perf_counter() - t0
    assert st == 0, st
    xg = x_gpu[sel]
    cell_bad = (xg.view(np.uint64) != res.x.view(np.uint64)).any(axis=1)
    g_bad = it_gpu[groups] != res.iters
    if res.rms is not None:
        g_bad |= np.asarray(rep.per_block_residual_rms)[groups].view(np.uint64) != res.rms.view(np.uint64)
        g_bad |= np.asarray(rep.per_block_flags)[groups] != res.flags
    den = np.maximum(np.abs(res.x).max(axis=1), 1e-300)
    rel = float((np.abs(xg - res.x).max(axis=1) / den).max())
    out = {"cells_checked": int(len(sel)), "groups_checked": int(len(groups)), "of_cells": int(cells),
           "mismatched_cells": int(cell_bad.sum()), "mismatched_groups": int(g_bad.sum()),
           "max_rel_err_x": rel, "max_iteration_diff": int(np.abs(it_gpu[groups] - res.iters).max()),
           "checker": checker, "checker_threads": threads, "checker_s": round(secs, 2),
           "compared": "x bits per cell; per-group iterations" + (", rms bits, flags" if res.rms is not None else "")}
    return out, (len(sel) / secs if len(sel) == cells else None), checker


def main_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2405_17363_b200 import Algo, BatchedSystem, DeviceSpec, Solver, Strategy
    from paper_2405_17363_b200.sharding import merge_reports, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = torch.cuda.device_count()
    shared_gpu = world > ngpu  # more ranks than GPUs (a smoke test of the N>1 path): ranks share devices
    local = local % ngpu
    torch.cuda.set_device(local)
    if world > 1:
        if shared_gpu:  # NCCL refuses two ranks on one device; gloo carries the barrier and the max
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    reg = regime(args.regime)
    algo = Algo.BICGSTAB_JACOBI if args.algo == "bicgstab" else Algo.BICG
    cfg = strategy_config(args.strategy)
    k = cfg.cells_per_block or (1024 // args.species if cfg.kind == Strategy.BlockCells else 1)
    replicas = cfg.kind == Strategy.MultiCells  # one global system: replicas only (sharding.py)
    n_total = args.cells * world  # weak scaling: every rank solves args.cells cells of the global batch
    if replicas:
        first, cells = 0, args.cells
    else:
        first, cells = shard_range(n_total, k, rank, world)  # contiguous, group-aligned ranges, no collectives
    m, h_values, h_rhs = make_workload(cells, first, args.cells if replicas else n_total, reg, args.species)
    nnz, n = m.nnz, m.species

    solver = Solver(local)
    stream = torch.cuda.current_stream()
    d_values = torch.from_numpy(h_values).cuda()
    d_rhs = torch.from_numpy(h_rhs).cuda()
    d_x = torch.empty((cells, n), dtype=torch.float64, device="cuda")
    dsys = BatchedSystem(n, cells, m.row_ptr, m.col_idx, d_values, d_rhs)
    dev = DeviceSpec()

    def step(timing=False, a=algo):
        return solver.run_strategy(dsys, cfg, dev, reg.tol, reg.max_iter, 1, a, stream=stream.cuda_stream,
                                   timing=timing, x_out=d_x)

    first_call_s = None
    for w in range(args.warmup):
        t0 = time.perf_counter()
        rep = step()
        if w == 0:  # includes building the schedule (annealing), once per pattern per process
            torch.cuda.synchronize()
            first_call_s = time.perf_counter() - t0
    launches0 = solver.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms, reports = [], []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            ev[i][0].record(stream)
            rep = step(timing=True)
            ev[i][1].record(stream)
            kernel_ms.append(rep.device_ms)
            reports.append(rep)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    barrier()
    launches = solver.kernel_launches - launches0
    x_timed = d_x.cpu().numpy()  # the last timed step's solution, for the parity check below
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(sum(step_ms))
    value = n_total * args.steps / (total_ms / 1e3)
    rep = reports[-1]
    iters = np.asarray(rep.per_block_iterations)
    merged = merge_reports(dict(iterations_effective=rep.iterations_effective, max_residual_rms=rep.max_residual_rms,
                                iterations_sum=rep.iterations_sum, breakdown_fallbacks=rep.breakdown_fallbacks,
                                n_groups=len(rep.per_block_iterations)))
    # it_c of every cell = its group's iteration count
    sizes = np.full(len(iters), cells // max(len(iters), 1), dtype=np.int64)
    if cfg.kind == Strategy.BlockCells and len(iters) > 1:
        sizes[:] = k
        sizes[-1] = cells - k * (len(iters) - 1)
    cell_iters = np.repeat(iters, sizes)
    alg_bytes = algorithmic_bytes(cell_iters, n, nnz)  # per launch (one solve of the rank's cells)
    kmean = statistics.mean(kernel_ms)
    achieved = alg_bytes / (kmean / 1e3) / 1e9
    peak, peak_kind = measured_peak_hbm()
    compulsory = cells * (8 * nnz + 16 * n + 16)
    kname = dominant_kernel(rep.kernels)
    clocks = clk.summary()
    tr = ncu_traffic()
    if not tr or tr.get("kernel") != kname or tr.get("cells") != cells or tr.get("species", 156) != n \
            or tr.get("algorithm", "bicgstab") != args.algo:
        tr = None  # the committed ncu capture is for another workload
    flops_per_it = (4 * nnz + 24 * n) if algo == Algo.BICGSTAB_JACOBI else (4 * nnz + 21 * n)
    fp64 = float(cell_iters.sum()) * flops_per_it / (kmean / 1e3) / 1e12
    # the binding resource, from this run: the planner's bank-model wavefronts
    # per group-iteration x the group-iterations / (SMs x SM clock x kernel time)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    smem_model = None
    if rep.model_spmv_wavefronts > 0 and clocks.get("sm_mhz"):
        wf = rep.model_spmv_wavefronts * float(iters.sum())
        smem_model = wf / (sms * clocks["sm_mhz"] * 1e6 * kmean / 1e3)

    # e2e through the public API with pinned host inputs
    e2e = None
    if not args.no_e2e:
        hsys = BatchedSystem(n, cells, m.row_ptr, m.col_idx, h_values, h_rhs)
        hx = torch.empty((cells, n), dtype=torch.float64, pin_memory=True).numpy()
        for _ in range(1):
            solver.run_strategy(hsys, cfg, dev, reg.tol, reg.max_iter, 1, algo, stream=stream.cuda_stream, x_out=hx)
        e_steps = max(1, min(args.steps, 5))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            r2 = solver.run_strategy(hsys, cfg, dev, reg.tol, reg.max_iter, 1, algo, stream=stream.cuda_stream,
                                     x_out=hx)
        torch.cuda.synchronize()
        e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3)
        barrier()
        ng = len(r2.per_block_iterations)
        e2e = {"value": n_total * e_steps / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h_values.nbytes + h_rhs.nbytes),
               "d2h_bytes_per_step": int(hx.nbytes + ng * (4 + 8 + 1)), "steps": e_steps,
               "ms_per_step": e_ms / e_steps}

    # end to end through the reference's own C++ entry point (blockcells::run_strategy
    # on the drop-in shim, a BatchedSystem of per-cell CsrMatrix/DenseVector)
    dropin = None
    exe = os.path.join(ROOT, "tests", "cpp", "bin", "dropin_bench")
    if rank == 0 and world == 1 and not args.no_dropin and os.path.exists(exe) and \
            cfg.kind == Strategy.BlockCells and cfg.cells_per_block == 1:
        env = dict(os.environ, BLOCKCELLS_B200_DEVICE=str(local))
        if args.algo == "bicgstab":
            env["BLOCKCELLS_B200_ALGO"] = "bicgstab"
        try:
            r = subprocess.run([exe, str(cells), str(max(1, min(args.steps, 5))), "1", str(n), repr(reg.h),
                                repr(reg.tol), str(reg.max_iter)], env=env, capture_output=True, text=True,
                               timeout=900)
            if r.returncode == 0:
                dropin = json.loads(r.stdout.strip().splitlines()[-1])
                dropin["h2d_bytes_per_step"] = dropin.pop("input_bytes_per_step")
                dropin["d2h_bytes_per_step"] = int(cells * n * 8)
            else:
                dropin = {"error": r.stderr[-300:]}
        except Exception as exc:  # the measurement is optional; its absence is reported
            dropin = {"error": str(exc)[:300]}

    # the reference's own algorithm on the GPU, same cells: a like-for-like
    # companion to the stock reference's BiCG number
    companion = None
    if algo == Algo.BICGSTAB_JACOBI and not args.no_companion:
        step(a=Algo.BICG)
        c_steps = 3
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(c_steps):
            rc = step(a=Algo.BICG)
        e1.record(stream)
        torch.cuda.synchronize()
        c_ms = max_over_ranks(e0.elapsed_time(e1))
        companion = {"value": n_total * c_steps / (c_ms / 1e3), "unit": UNIT, "steps": c_steps,
                     "ms_per_step": c_ms / c_steps, "algorithm": "bicg",
                     "iterations_sum": int(sum_over_ranks(rc.iterations_sum))}
        rep = reports[-1]

    # parity: the last timed step's output against the checker, bit for bit
    parity, cpu = None, None
    if not args.no_parity:
        rep.per_cell_x = x_timed
        threads = max(1, (os.cpu_count() or 1) // (world if not shared_gpu else world))
        budget = cells if world == 1 else max(1, args.parity_cells // world)
        budget = min(budget, args.parity_cells)
        parity, all_rate, checker = parity_check(args, rep, m, h_values, h_rhs, reg, ref_strategy(args.strategy),
                                                 k, budget, threads)
        for key in ("cells_checked", "mismatched_cells", "mismatched_groups", "groups_checked"):
            parity[key] = int(sum_over_ranks(parity[key]))
        parity["max_rel_err_x"] = max_over_ranks(parity["max_rel_err_x"])
        if rank == 0 and world == 1 and all_rate:
            cpu = {"value": all_rate, "unit": UNIT, "cores": threads,
                   "kind": "reference" if "oracle/_ref" in checker else "port",
                   "sample": f"{checker}: all {cells} cells of the workload (the parity run), {threads} threads"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        code = ref_strategy(args.strategy)
        if cpu is None:
            rate, cores, sample, kind = cpu_reference_rate(h_values, h_rhs, m.row_ptr, m.col_idx, reg,
                                                           args.cpu_seconds, args.algo, cfg_code=code)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
        # BASELINE.json configs[1]: the reference on one host thread as well
        rate1, _, sample1, kind1 = cpu_reference_rate(h_values, h_rhs, m.row_ptr, m.col_idx, reg,
                                                      max(2.0, args.cpu_seconds / 3), args.algo, threads=1,
                                                      cfg_code=code)
        cpu["single_thread"] = {"value": rate1, "unit": UNIT, "cores": 1, "kind": kind1, "sample": sample1}
        if args.algo == "bicgstab":  # the reference's stock algorithm (BiCG run_strategy), all cores
            rate_b, cores_b, sample_b, kind_b = cpu_reference_rate(h_values, h_rhs, m.row_ptr, m.col_idx, reg,
                                                                   args.cpu_seconds, "bicg", cfg_code=code)
            cpu["reference_bicg"] = {"value": rate_b, "unit": UNIT, "cores": cores_b, "kind": kind_b,
                                     "sample": sample_b}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, n, nnz, cells, n_total, reg, world),
            "solve": {"iterations_sum": int(merged["iterations_sum"]),
                      "breakdown_fallbacks": int(merged["breakdown_fallbacks"]),
                      "ranks_share_gpus": bool(shared_gpu),
                      "first_call_s": first_call_s,
                      "first_call_is": "wall time of the first (warm-up) solve: schedule planning for the pattern "
                                       "(simulated annealing, once per pattern and process) plus one solve"},
            "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": (tr or {}).get("dram_bytes_per_launch_scaled"),
                         "kernel": kname, "kernel_ms": kmean, "algorithmic_bytes": alg_bytes,
                         "peak_kind": peak_kind,
                         "frac_is": "SURVEY.md 8d streaming-HBM bytes / HBM peak (the metric's label); the "
                                    "kernel keeps the per-iteration bytes on chip, so the bound is the "
                                    "shared-memory pipe (binding)",
                         "compulsory_bytes": compulsory,
                         "compulsory_frac": compulsory / (kmean / 1e3) / 1e9 / peak,
                         "fp64_tflops": fp64,
                         "binding": {
                             "resource": "shared-memory LSU pipe (wavefronts)",
                             "frac_model": smem_model,
                             "model_wavefronts_per_group_iteration": rep.model_spmv_wavefronts,
                             "frac_model_is": "planner bank-model SpMV wavefronts x group-iterations / "
                                              "(SMs x measured SM clock x kernel time), this run",
                             "frac_ncu": (tr or {}).get("shared_pipe_frac"),
                             "issue_active_frac_ncu": (tr or {}).get("issue_active_frac"),
                             "fp64_pipe_frac_ncu": (tr or {}).get("fp64_pipe_frac"),
                             "ncu_source": f"profiles/ncu_block_cells_traffic.json tag {tr.get('tag')}" if tr else None}},
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_dropin": dropin,
            "bicg_companion": companion,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "wall_s_timed": t_wall,
        }
        print(json.dumps(out), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        main_reference(args)
    else:
        main_b200(args)


if __name__ == "__main__":
    main()
