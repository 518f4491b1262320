"""The reference's benchmark layer (bench.hpp, bench.cpp) over the device
simulation: SURVEY.md §8f rank 4.

``run_experiment`` runs every configured strategy through the device-resident
``simulate.run_simulation`` (bc_simulate) on the same generated problem and
aggregates per-step records exactly as bench.cpp:94-187 does (two-pass
mean/population std, speedup against the one-cell baseline, iteration ratio
against block-cells(1)).  ``to_csv`` / ``emit_csv`` write results.csv with
bench.cpp's exact header and std::to_chars shortest round-trip reals;
``summary_to_json`` / ``emit_summary_json`` write summary.json with
bench.cpp's key order and nlohmann::json's number formatting, so the
reference's ``parse_csv`` and ``summary_stats_from_json`` read GPU runs
back (tests/test_experiment.py checks both against oracle/_ref).

The summary's kernel_plan / occupancy / memory fields are the reference's
analytic GPU model (exec_model.cpp:102-200), restated here because the
schema carries them; each strategy additionally gets a "b200" object with
what actually ran (kernels, launches, device time).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from decimal import Decimal
from typing import List, Optional

from .simulate import LinearSolverChoice, SimulationConfig, run_simulation
from .solver import Algo, DeviceSpec, Strategy, StrategyConfig, UnsupportedMechanism, InvalidGrouping
from .workload import IDEAL, REALISTIC, Mechanism

CSV_HEADER = ("step,strategy,cells,species,cells_per_block,iterations_effective,"
              "iterations_sum,wall_ns,max_residual_rms,breakdown_fallbacks,clip_events")
PAPER_AUX_ARRAYS = 9          # bench.cpp:22
ACTUAL_AUX_ARRAYS = 6         # BicgWorkspace::aux_array_count() (bicg.hpp:22)
STRATEGY_NAMES = {Strategy.OneCell: "one-cell", Strategy.MultiCells: "multi-cells", Strategy.BlockCells: "block-cells"}


# --- number formatting -----------------------------------------------------------

def _digits(v: float):
    """Shortest round-trip decimal digits and the decimal point position n
    (value = 0.d1d2... * 10^n), as repr / grisu / Ryu produce them."""
    t = Decimal(repr(abs(v))).normalize().as_tuple()
    ds = "".join(map(str, t.digits))
    return ds, len(ds) + t.exponent


def format_double(v: float) -> str:
    """std::to_chars(double) (format.cpp:9-14): the shorter of fixed and
    scientific (exponent at least two digits), fixed on a tie."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    ds, n = _digits(v)
    k = len(ds)
    if n >= k:  # integral: to_chars prints the exact integer in fixed form
        fixed = str(int(abs(v)))
    elif n > 0:
        fixed = ds[:n] + "." + ds[n:]
    else:
        fixed = "0." + "0" * (-n) + ds
    e = n - 1
    sci = ds[0] + ("." + ds[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def _json_double(v: float) -> str:
    """nlohmann::json's dump of a double (dtoa_impl::format_buffer with
    min_exp -4, max_exp 15): digits[000].0, dig.its, 0.[000]digits or
    d[.igits]e+XX."""
    if not math.isfinite(v):
        return "null"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0.0"
    ds, n = _digits(v)
    k = len(ds)
    if k <= n <= 15:
        body = ds + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        body = ds[:n] + "." + ds[n:]
    elif -4 < n <= 0:
        body = "0." + "0" * (-n) + ds
    else:
        e = n - 1
        body = ds[0] + ("." + ds[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    return sign + body


def _dump(obj, indent=2, level=0) -> str:
    """nlohmann::ordered_json::dump(2): insertion-ordered keys, doubles per
    _json_double, integers as integers."""
    pad, inner = " " * (indent * level), " " * (indent * (level + 1))
    if obj is None:
        return "null"
    if obj is True or obj is False:
        return "true" if obj else "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return _json_double(obj)
    if isinstance(obj, str):
        return json.dumps(obj, ensure_ascii=False)
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [f"{inner}{json.dumps(k)}: {_dump(v, indent, level + 1)}" for k, v in obj.items()]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(obj, (list, tuple)):
        if not obj:
            return "[]"
        return "[\n" + ",\n".join(inner + _dump(v, indent, level + 1) for v in obj) + "\n" + pad + "]"
    raise TypeError(type(obj))


# --- the reference's analytic GPU model (exec_model.cpp:90-200) ---------------------

def next_pow2(n: int) -> int:
    if n < 1:
        raise ValueError("next_pow2: n must be >= 1")
    return 1 << (n - 1).bit_length()


@dataclass
class KernelPlan:
    strategy: Strategy = Strategy.OneCell
    cells_per_block: float = 1.0
    threads_per_block: int = 0
    shared_slots: int = 0
    full_blocks: int = 0
    remainder: Optional[dict] = None  # {"cells", "threads", "shared_slots"}

    def total_blocks(self) -> int:
        return self.full_blocks + (1 if self.remainder else 0)

    def to_json_obj(self):
        return {"strategy": STRATEGY_NAMES[self.strategy], "cells_per_block": float(self.cells_per_block),
                "threads_per_block": self.threads_per_block, "shared_slots": self.shared_slots,
                "full_blocks": self.full_blocks, "remainder": self.remainder}


def plan_kernel(strategy: Strategy, total_cells: int, species: int, device: DeviceSpec = DeviceSpec(),
                k_request: Optional[int] = None) -> KernelPlan:
    """exec_model.cpp:102-161."""
    if total_cells < 1:
        raise ValueError("plan_kernel: total_cells must be >= 1")
    if species < 1:
        raise ValueError("plan_kernel: species must be >= 1")
    mtpb = device.max_threads_per_block
    if species > mtpb:
        raise UnsupportedMechanism("mechanism needs more threads per cell than a block provides")
    p = KernelPlan(strategy=strategy)
    if strategy == Strategy.OneCell:
        p.cells_per_block, p.threads_per_block = 1.0, species
        p.shared_slots, p.full_blocks = next_pow2(species), total_cells
    elif strategy == Strategy.MultiCells:
        p.threads_per_block, p.shared_slots = mtpb, next_pow2(mtpb)
        p.cells_per_block = mtpb / species
        p.full_blocks = (total_cells * species + mtpb - 1) // mtpb
    else:
        if k_request is not None:
            k = int(k_request)
            if k < 1:
                raise ValueError("plan_kernel: cells per block must be >= 1")
            if k * species > mtpb:
                raise InvalidGrouping("requested cells per block exceeds the thread budget")
        else:
            k = mtpb // species
        p.cells_per_block, p.threads_per_block = float(k), k * species
        p.shared_slots, p.full_blocks = next_pow2(k * species), total_cells // k
        left = total_cells % k
        if left:
            p.remainder = {"cells": left, "threads": left * species, "shared_slots": next_pow2(left * species)}
    return p


def occupancy_estimate(plan: KernelPlan, device: DeviceSpec = DeviceSpec()):
    """exec_model.cpp:163-185: (value, shared_mem_exceeded)."""
    warps = (plan.threads_per_block + device.warp_size - 1) // device.warp_size
    padded = warps * device.warp_size
    shared = plan.shared_slots * device.shared_slot_bytes
    if shared > device.shared_mem_per_sm or padded > device.max_threads_per_sm:
        return 0.0, shared > device.shared_mem_per_sm
    blocks = min(device.max_blocks_per_sm, device.max_threads_per_sm // padded, device.shared_mem_per_sm // shared)
    return min(blocks * warps / device.max_warps_per_sm, 1.0), False


def memory_estimate(strategy: Strategy, cells: int, species: int, aux: int, device: DeviceSpec = DeviceSpec(),
                    k_request: Optional[int] = None) -> int:
    """exec_model.cpp:187-200."""
    plan = plan_kernel(strategy, cells, species, device, k_request)
    b = (2 + aux) * cells * species * 8 + plan.total_blocks() * 8
    if strategy == Strategy.MultiCells:
        b += 2 * cells * 8
    return b


# --- bench.hpp ------------------------------------------------------------------------

@dataclass
class ExperimentConfig:
    """bench.hpp:17-37 (+ the linear-solver algorithm)."""
    cells: int = 1000
    species: int = 156
    steps: int = 720
    dt_seconds: float = 120.0
    mode: int = REALISTIC
    strategies: List[StrategyConfig] = field(default_factory=list)
    tol: float = 1e-30
    max_iter: int = 1000
    seed: int = 0
    worker_count: int = 1
    output_path: str = ""
    device: DeviceSpec = field(default_factory=DeviceSpec)
    algo: Algo = Algo.BICG

    def n_reactions(self) -> int:
        return 3 * self.species

    def check(self) -> None:  # bench.cpp:69-78
        if self.cells < 1:
            raise ValueError("experiment: cells must be >= 1")
        if self.species < 2:
            raise ValueError("experiment: species must be >= 2")
        if not self.dt_seconds > 0.0:
            raise ValueError("experiment: dt must be positive")
        if not self.tol > 0.0:
            raise ValueError("experiment: tol must be positive")
        if self.max_iter < 1:
            raise ValueError("experiment: max_iter must be >= 1")
        if not self.strategies:
            raise ValueError("experiment: no strategies configured")


@dataclass
class StepRecord:
    """bench.hpp:39-53 (the CSV row, in column order)."""
    step: int = 0
    strategy: str = ""
    cells: int = 0
    species: int = 0
    cells_per_block: float = 0.0
    iterations_effective: int = 0
    iterations_sum: int = 0
    wall_ns: int = 0
    max_residual_rms: float = 0.0
    breakdown_fallbacks: int = 0
    clip_events: int = 0


@dataclass
class MeanStd:
    mean: float = 0.0
    std: float = 0.0


def mean_std(xs) -> MeanStd:
    """bench.cpp:80-91: two-pass mean and population std."""
    xs = [float(x) for x in xs]
    if not xs:
        return MeanStd()
    s = 0.0
    for x in xs:
        s += x
    m = s / len(xs)
    sq = 0.0
    for x in xs:
        sq += (x - m) * (x - m)
    return MeanStd(m, math.sqrt(sq / len(xs)))


@dataclass
class StrategyStats:
    config: StrategyConfig
    plan: KernelPlan
    occupancy: float
    occupancy_shared_mem_exceeded: bool
    memory_bytes_paper_census: int
    memory_bytes_actual_census: int
    iterations_effective: MeanStd
    wall_ns: MeanStd
    speedup_vs_baseline: Optional[float] = None
    iteration_reduction_vs_block1: Optional[MeanStd] = None
    b200: dict = field(default_factory=dict)


@dataclass
class ExperimentResult:
    per_strategy: List[StrategyStats] = field(default_factory=list)
    raw: List[StepRecord] = field(default_factory=list)
    final_states_per_strategy: list = field(default_factory=list)


def label(cfg: StrategyConfig) -> str:
    """strategies.cpp:109-119."""
    if cfg.kind == Strategy.BlockCells:
        return f"block-cells({cfg.cells_per_block})" if cfg.cells_per_block else "block-cells(N)"
    return STRATEGY_NAMES[Strategy(cfg.kind)]


def run_experiment(config: ExperimentConfig, solver=None) -> ExperimentResult:
    """bench.cpp:94-187 with every simulation on the GPU."""
    config.check()
    mech = Mechanism(config.species, config.n_reactions(), config.seed)
    result = ExperimentResult()
    iters_per, wall_per = [], []
    for strat in config.strategies:
        sim = SimulationConfig(cells=config.cells, mode=config.mode, steps=config.steps,
                               dt_seconds=config.dt_seconds, tol=config.tol, max_iter=config.max_iter,
                               worker_count=config.worker_count,
                               solver=LinearSolverChoice(False, strat, config.algo), device=config.device)
        sr = run_simulation(mech, sim, None, solver=solver)
        k = strat.cells_per_block if strat.kind == Strategy.BlockCells else None
        plan = plan_kernel(Strategy(strat.kind), config.cells, config.species, config.device, k)
        iters, wall = [], []
        for s in sr.per_step:
            result.raw.append(StepRecord(s.step, STRATEGY_NAMES[Strategy(strat.kind)], config.cells, config.species,
                                         plan.cells_per_block, s.iterations_effective, s.iterations_sum,
                                         s.wall_time_ns, s.max_residual_rms, s.breakdown_fallbacks, s.clip_events))
            iters.append(float(s.iterations_effective))
            wall.append(float(s.wall_time_ns))
        occ, exceeded = occupancy_estimate(plan, config.device)
        result.per_strategy.append(StrategyStats(
            config=strat, plan=plan, occupancy=occ, occupancy_shared_mem_exceeded=exceeded,
            memory_bytes_paper_census=memory_estimate(Strategy(strat.kind), config.cells, config.species,
                                                      PAPER_AUX_ARRAYS, config.device, k),
            memory_bytes_actual_census=memory_estimate(Strategy(strat.kind), config.cells, config.species,
                                                       ACTUAL_AUX_ARRAYS, config.device, k),
            iterations_effective=mean_std(iters), wall_ns=mean_std(wall),
            b200={"algorithm": Algo(config.algo).name.lower(), "device_resident": True}))
        result.final_states_per_strategy.append(sr.final_states)
        iters_per.append(iters)
        wall_per.append(wall)
    base = next((i for i, s in enumerate(config.strategies) if s.kind == Strategy.OneCell), -1)
    blk1 = next((i for i, s in enumerate(config.strategies)
                 if s.kind == Strategy.BlockCells and s.cells_per_block == 1), -1)
    for i, st in enumerate(result.per_strategy):
        if base >= 0 and st.wall_ns.mean > 0.0:
            st.speedup_vs_baseline = result.per_strategy[base].wall_ns.mean / st.wall_ns.mean
        if blk1 >= 0:
            ratios = [n / d for n, d in zip(iters_per[i], iters_per[blk1]) if d > 0.0]
            if ratios:
                st.iteration_reduction_vs_block1 = mean_std(ratios)
    return result


def to_csv(raw: List[StepRecord]) -> str:
    """bench.cpp:189-218."""
    if not raw:
        raise ValueError("emit_csv: empty table")
    lines = [CSV_HEADER]
    for r in raw:
        lines.append(",".join([str(r.step), r.strategy, str(r.cells), str(r.species), format_double(r.cells_per_block),
                               str(r.iterations_effective), str(r.iterations_sum), str(r.wall_ns),
                               format_double(r.max_residual_rms), str(r.breakdown_fallbacks), str(r.clip_events)]))
    return "\n".join(lines) + "\n"


def parse_csv(text: str) -> List[StepRecord]:
    """bench.cpp:229-256."""
    lines = text.split("\n")
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError("csv: missing or unexpected header")
    rows = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 11:
            raise ValueError(f"csv: expected 11 fields, got {len(f)}")
        rows.append(StepRecord(int(f[0]), f[1], int(f[2]), int(f[3]), float(f[4]), int(f[5]), int(f[6]), int(f[7]),
                               float(f[8]), int(f[9]), int(f[10])))
    return rows


def _strategy_json(cfg: StrategyConfig):
    j = {"kind": STRATEGY_NAMES[Strategy(cfg.kind)]}
    if cfg.kind == Strategy.BlockCells:
        j["cells_per_block"] = int(cfg.cells_per_block) if cfg.cells_per_block else "N"
    return j


def summary_to_json(config: ExperimentConfig, stats: List[StrategyStats]) -> str:
    """bench.cpp:285-330 (key order kept)."""
    if not stats:
        raise ValueError("emit_summary_json: no strategies")
    jc = {"cells": config.cells, "species": config.species, "steps": config.steps,
          "dt_seconds": float(config.dt_seconds), "mode": "ideal" if config.mode == IDEAL else "realistic",
          "strategies": [_strategy_json(s) for s in config.strategies], "tol": float(config.tol),
          "max_iter": config.max_iter, "seed": config.seed, "worker_count": config.worker_count,
          "output_path": config.output_path}
    js = []
    for s in stats:
        ms = lambda m: {"mean": float(m.mean), "std": float(m.std)}  # noqa: E731
        js.append({"label": label(s.config), "config": _strategy_json(s.config), "kernel_plan": s.plan.to_json_obj(),
                   "occupancy": float(s.occupancy), "occupancy_shared_mem_exceeded": bool(s.occupancy_shared_mem_exceeded),
                   "memory_bytes_paper_census": s.memory_bytes_paper_census,
                   "memory_bytes_actual_census": s.memory_bytes_actual_census,
                   "iterations_effective": ms(s.iterations_effective), "wall_ns": ms(s.wall_ns),
                   "speedup_vs_baseline": None if s.speedup_vs_baseline is None else float(s.speedup_vs_baseline),
                   "iteration_reduction_vs_block1": None if s.iteration_reduction_vs_block1 is None
                   else ms(s.iteration_reduction_vs_block1),
                   **({"b200": s.b200} if s.b200 else {})})
    return _dump({"config": jc, "strategies": js})


def emit_csv(raw: List[StepRecord], path: str) -> None:
    with open(path, "w", newline="\n") as f:
        f.write(to_csv(raw))


def emit_summary_json(config: ExperimentConfig, stats: List[StrategyStats], path: str) -> None:
    with open(path, "w", newline="\n") as f:
        f.write(summary_to_json(config, stats) + "\n")


def write_outputs(config: ExperimentConfig, result: ExperimentResult) -> None:
    """results.csv + summary.json under config.output_path (as the reference's driver does)."""
    os.makedirs(config.output_path, exist_ok=True)
    emit_csv(result.raw, os.path.join(config.output_path, "results.csv"))
    emit_summary_json(config, result.per_strategy, os.path.join(config.output_path, "summary.json"))
