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
  roofline  dominant kernel (block_cells_kernel): algorithmic streaming bytes
            (it*(16*nnz+80*n)+16*n+16 per cell) / its event time,
            against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference's own solver (oracle/_ref, run_strategy
            Block-cells(1), all host threads) on a bounded sample, rank 0, N=1

  --impl reference   times the reference's CPU implementation only.
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


def cpu_reference_rate(values, rhs, row_ptr, col_idx, reg, budget_s, algo_name="bicg", threads=None):
    """The reference's run_strategy (Block-cells(1), all host threads unless
    `threads`) on a bounded prefix sample of the workload.  Returns (rate,
    cores, sample, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as of
    cores = threads or os.cpu_count() or 1
    use_ref = of.have_ref() and algo_name == "bicg"
    kind = "reference" if use_ref else "port"

    def run(nc):
        """Seconds of solver time: SolveReport::wall_time_ns for the reference
        (the whole run_strategy call, strategies.cpp:241-247), wall clock for the port."""
        if use_ref:
            st, res = of.ref_solve_batch(2, 1, row_ptr, col_idx, values[:nc], rhs[:nc], reg.tol, reg.max_iter,
                                         workers=cores)
            assert st == 0, st
            return res.report.wall_time_ns / 1e9
        else:
            st, res = of.orc_solve_batch(2, 0 if algo_name == "bicg" else 1, 1, row_ptr, col_idx, values[:nc],
                                         rhs[:nc], reg.tol, reg.max_iter, workers=cores)
            assert st == 0, st
            return None

    probe = min(len(values), 4 * cores)
    t0 = time.perf_counter()
    dt = run(probe) or (time.perf_counter() - t0)
    nc = int(min(len(values), max(probe, probe * budget_s / max(dt, 1e-3))))
    t0 = time.perf_counter()
    dt = run(nc) or (time.perf_counter() - t0)
    solver = "reference run_strategy Block-cells(1) BiCG" if use_ref else f"oracle port {algo_name}"
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


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    reg = regime(args.regime)
    n_total = args.cells * args.gpus
    m, values, rhs = make_workload(min(args.cells, 50_000), 0, n_total, reg, args.species)
    budget = max(2.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    rates = []
    for i in range(args.warmup + args.steps):
        rate, cores, sample, kind = cpu_reference_rate(values, rhs, m.row_ptr, m.col_idx, reg, budget)
        if i >= args.warmup:
            rates.append(rate)
    value = statistics.median(rates)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * args.cells / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"M{args.species}, {args.cells} cells/GPU, Block-cells(1), {reg.name} regime; reference CPU "
                               "solver (unpreconditioned BiCG, its only algorithm) on bounded samples",
                   "algorithm": "bicg (reference)", "regime": reg.name},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


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

    reg = regime(args.regime)
    algo = Algo.BICGSTAB_JACOBI if args.algo == "bicgstab" else Algo.BICG
    cfg = strategy_config(args.strategy)
    k = cfg.cells_per_block or (1024 // args.species if cfg.kind == Strategy.BlockCells else 1)
    n_total = args.cells * world  # weak scaling: every rank solves args.cells cells of the global batch
    first, cells = shard_range(n_total, k, rank, world)  # contiguous, group-aligned ranges, no collectives
    m, h_values, h_rhs = make_workload(cells, first, n_total, reg, args.species)
    nnz, n = m.nnz, m.species

    solver = Solver(local)
    stream = torch.cuda.current_stream()
    d_values = torch.from_numpy(h_values).cuda()
    d_rhs = torch.from_numpy(h_rhs).cuda()
    d_x = torch.empty((cells, n), dtype=torch.float64, device="cuda")
    dsys = BatchedSystem(n, cells, m.row_ptr, m.col_idx, d_values, d_rhs)
    dev = DeviceSpec()

    def step(timing=False):
        return solver.run_strategy(dsys, cfg, dev, reg.tol, reg.max_iter, 1, algo, stream=stream.cuda_stream,
                                   timing=timing, x_out=d_x)

    for _ in range(args.warmup):
        rep = step()
    launches0 = solver.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms, iters_total, reports = [], 0, []
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
    tr = ncu_traffic()
    if not tr or tr.get("kernel") != kname or tr.get("cells") != cells or tr.get("species", 156) != n:
        tr = None  # the committed ncu capture is for another workload
    flops_per_it = (4 * nnz + 24 * n) if algo == Algo.BICGSTAB_JACOBI else (4 * nnz + 21 * n)
    fp64 = float(cell_iters.sum()) * flops_per_it / (kmean / 1e3) / 1e12

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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, sample, kind = cpu_reference_rate(h_values, h_rhs, m.row_ptr, m.col_idx, reg, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
        # BASELINE.json configs[1]: the reference on one host thread as well
        rate1, _, sample1, kind1 = cpu_reference_rate(h_values, h_rhs, m.row_ptr, m.col_idx, reg,
                                                      max(2.0, args.cpu_seconds / 3), threads=1)
        cpu["single_thread"] = {"value": rate1, "unit": UNIT, "cores": 1, "kind": kind1, "sample": sample1}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": (f"M{n} ({n} species, {nnz} nnz) first Newton system of step 0, {cells} cells/GPU "
                             f"({n_total} total), {args.strategy}, {'Jacobi-BiCGSTAB' if algo else 'BiCG'}, "
                             f"{reg.name} regime (h={reg.h:g} s, tol={reg.tol:g}, max_iter={reg.max_iter})"),
                "cells_per_gpu": cells, "global_cells": n_total, "strategy": args.strategy,
                "algorithm": args.algo, "regime": reg.name, "iterations_sum": int(merged["iterations_sum"]),
                "breakdown_fallbacks": int(merged["breakdown_fallbacks"]),
                "l2": f"inputs larger than L2 ({h_values.nbytes / 1e9:.3f} GB values per GPU vs 126 MB L2)",
                "parallelism": f"cell-range sharding over {world} GPU(s), no collectives"
                               + (f" ({world} ranks sharing {ngpu} GPU(s): a test of the N>1 path, not a"
                                  " scaling number)" if shared_gpu else ""),
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": (tr or {}).get("dram_bytes_per_launch_scaled"),
                         "kernel": kname, "kernel_ms": kmean, "algorithmic_bytes": alg_bytes,
                         "peak_kind": peak_kind,
                         "compulsory_bytes": compulsory,
                         "compulsory_frac": compulsory / (kmean / 1e3) / 1e9 / peak,
                         "fp64_tflops": fp64,
                         # what actually binds the kernel (ncu --set full of the same workload, profiles/):
                         # the per-iteration bytes never leave the SM, so HBM is not it
                         "measured_bound": None if not tr else {
                             "resource": "shared-memory pipe (LSU wavefronts)", "frac": tr.get("shared_pipe_frac"),
                             "issue_active_frac": tr.get("issue_active_frac"),
                             "fp64_pipe_frac": tr.get("fp64_pipe_frac"), "source": f"ncu tag {tr.get('tag')}"}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
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
