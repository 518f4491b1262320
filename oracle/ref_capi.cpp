// ref_capi.cpp -- flat C entry points over the UNMODIFIED reference library,
// compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libbcref.so.  TEST INFRASTRUCTURE ONLY: used by tests/ to pin
// the C restatement (bc_oracle.c) and the CUDA path, and by bench.py's
// reference arm / cpu_baseline leg.  No reference source is copied here; this
// file only converts plain arrays to the reference's types and calls its
// public API (strategies.hpp:60-82, bicg.hpp:42-48, dense_lu.hpp:28-33,
// mechanism.hpp:45-125, simulate.hpp:29-32, bench.hpp:69-104, format.hpp).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "blockcells/bench.hpp"
#include "blockcells/bicg.hpp"
#include "blockcells/format.hpp"
#include "blockcells/dense_lu.hpp"
#include "blockcells/exec_model.hpp"
#include "blockcells/mechanism.hpp"
#include "blockcells/reduction.hpp"
#include "blockcells/simulate.hpp"
#include "blockcells/strategies.hpp"

using namespace blockcells;

namespace {

int map_exception() {
    try {
        throw;
    } catch (const InvalidGrouping&) {
        return -2;
    } catch (const UnsupportedMechanism&) {
        return -3;
    } catch (const SingularMatrix&) {
        return -4;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::bad_alloc&) {
        return -7;
    } catch (...) {
        return -8;
    }
}

CsrMatrix make_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* va) {
    CsrMatrix m;
    m.n_rows = m.n_cols = static_cast<std::size_t>(n);
    m.row_ptr.assign(rp, rp + n + 1);
    m.col_idx.assign(ci, ci + rp[n]);
    m.values.assign(va, va + rp[n]);
    return m;
}

}  // namespace

extern "C" {

typedef struct {
    int64_t n_groups;
    int64_t iterations_effective;
    int64_t iterations_sum;
    double max_residual_rms;
    int64_t breakdown_fallbacks;
    double cells_per_block;
    int64_t wall_time_ns;
} ref_report;

// run_strategy (strategies.cpp:251-264) on a batch sharing one pattern.
// strategy: 0 one-cell, 1 multi-cells, 2 block-cells; k_request 0 = "N".
int ref_solve_batch(int strategy, int64_t k_request, int64_t species, int64_t cells,
                    const int32_t* row_ptr, const int32_t* col_idx, const double* values,
                    const double* rhs, double tol, int64_t max_iter,
                    int64_t max_threads_per_block, int64_t workers, double* x_out,
                    int64_t* group_iters, ref_report* report) {
    try {
        BatchedSystem sys;
        sys.species = static_cast<std::size_t>(species);
        sys.cells = static_cast<std::size_t>(cells);
        const int64_t nnz = row_ptr[species];
        CsrMatrix proto;
        proto.n_rows = proto.n_cols = sys.species;
        proto.row_ptr.assign(row_ptr, row_ptr + species + 1);
        proto.col_idx.assign(col_idx, col_idx + nnz);
        sys.per_cell_matrices.reserve(sys.cells);
        sys.per_cell_rhs.reserve(sys.cells);
        for (int64_t c = 0; c < cells; ++c) {
            CsrMatrix m = proto;
            m.values.assign(values + c * nnz, values + (c + 1) * nnz);
            sys.per_cell_matrices.push_back(std::move(m));
            sys.per_cell_rhs.emplace_back(rhs + c * species, rhs + (c + 1) * species);
        }
        StrategyConfig cfg;
        cfg.kind = strategy == 0 ? Strategy::OneCell
                   : strategy == 1 ? Strategy::MultiCells
                                   : Strategy::BlockCells;
        if (k_request > 0) cfg.cells_per_block = static_cast<std::size_t>(k_request);
        DeviceSpec dev;
        dev.max_threads_per_block = static_cast<std::size_t>(max_threads_per_block);
        if (dev.max_threads_per_sm < dev.max_threads_per_block)
            dev.max_threads_per_sm = dev.max_threads_per_block;
        const SolveReport rep = run_strategy(sys, cfg, dev, tol,
                                             static_cast<std::size_t>(max_iter),
                                             static_cast<std::size_t>(workers));
        for (int64_t c = 0; c < cells; ++c)
            std::memcpy(x_out + c * species, rep.per_cell_x[c].data(),
                        sizeof(double) * species);
        if (group_iters)
            for (std::size_t g = 0; g < rep.per_block_iterations.size(); ++g)
                group_iters[g] = static_cast<int64_t>(rep.per_block_iterations[g]);
        if (report) {
            report->n_groups = static_cast<int64_t>(rep.per_block_iterations.size());
            report->iterations_effective = static_cast<int64_t>(rep.iterations_effective);
            report->iterations_sum = static_cast<int64_t>(rep.iterations_sum);
            report->max_residual_rms = rep.max_residual_rms;
            report->breakdown_fallbacks = static_cast<int64_t>(rep.breakdown_fallbacks);
            report->cells_per_block = rep.cells_per_block;
            report->wall_time_ns = rep.wall_time_ns;
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// bicg_solve (bicg.cpp:42-142) with an explicit ReductionPlan.
int ref_bicg_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                   const double* b, const double* x0, double tol, int64_t max_iter,
                   const int64_t* ranges /* pairs */, int64_t n_blocks, int host_stage,
                   double* x_out, int64_t* iterations, double* rms, int32_t* converged,
                   int32_t* breakdown) {
    try {
        const CsrMatrix a = make_csr(n, rp, ci, va);
        ReductionPlan plan;
        for (int64_t k = 0; k < n_blocks; ++k)
            plan.block_ranges.push_back({static_cast<std::size_t>(ranges[2 * k]),
                                         static_cast<std::size_t>(ranges[2 * k + 1])});
        plan.host_stage = host_stage != 0;
        const SolveOutcome out = bicg_solve(a, DenseVector(b, b + n), DenseVector(x0, x0 + n),
                                            tol, static_cast<std::size_t>(max_iter), plan);
        std::memcpy(x_out, out.x.data(), sizeof(double) * n);
        *iterations = static_cast<int64_t>(out.iterations);
        *rms = out.final_residual_rms;
        *converged = out.converged;
        *breakdown = out.breakdown;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// lu_solve (dense_lu.cpp:65-67).
int ref_lu_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                 const double* b, double* x_out) {
    try {
        const DenseVector x = lu_solve(make_csr(n, rp, ci, va), DenseVector(b, b + n));
        std::memcpy(x_out, x.data(), sizeof(double) * n);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// tree_reduce (reduction.cpp:46-51) and plan_reduce (reduction.cpp:53-58).
double ref_tree_reduce(const double* v, int64_t len, int64_t padded) {
    return tree_reduce(std::span<const double>(v, static_cast<std::size_t>(len)),
                       static_cast<std::size_t>(padded));
}

double ref_plan_reduce(const double* v, int64_t n, const int64_t* ranges, int64_t n_blocks) {
    ReductionPlan plan;
    for (int64_t k = 0; k < n_blocks; ++k)
        plan.block_ranges.push_back({static_cast<std::size_t>(ranges[2 * k]),
                                     static_cast<std::size_t>(ranges[2 * k + 1])});
    plan.host_stage = n_blocks > 1;
    return plan_reduce(std::span<const double>(v, static_cast<std::size_t>(n)), plan);
}

// Pattern of the synthetic mechanism (mechanism.cpp:117-150, 172-219).
// Call with row_ptr/col_idx NULL to query nnz.
int ref_mechanism_pattern(int64_t species, int64_t reactions, uint64_t seed, int64_t* nnz,
                          int32_t* row_ptr, int32_t* col_idx) {
    try {
        const MechanismEvaluator ev(generate_mechanism(static_cast<std::size_t>(species),
                                                       static_cast<std::size_t>(reactions), seed));
        const CsrMatrix& p = ev.pattern();
        *nnz = static_cast<int64_t>(p.nnz());
        if (row_ptr)
            for (std::size_t i = 0; i <= p.n_rows; ++i) row_ptr[i] = static_cast<int32_t>(p.row_ptr[i]);
        if (col_idx)
            for (std::size_t j = 0; j < p.nnz(); ++j) col_idx[j] = static_cast<int32_t>(p.col_idx[j]);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// The first Newton system of step 0 for cells [first, first+count) of a
// total_cells batch: newton_system(M, cell_conditions(c, C, mode), y=1,
// y_prev=1, h) (simulate.cpp:46-64).  mode: 0 ideal, 1 realistic.
int ref_newton_batch(int64_t species, int64_t reactions, uint64_t seed, int64_t first,
                     int64_t count, int64_t total_cells, int mode, double h, double* values,
                     double* rhs) {
    try {
        const MechanismSpec mech = generate_mechanism(static_cast<std::size_t>(species),
                                                      static_cast<std::size_t>(reactions), seed);
        const CellState ones{DenseVector(static_cast<std::size_t>(species), 1.0)};
        for (int64_t c = 0; c < count; ++c) {
            const CellConditions cond = cell_conditions(
                static_cast<std::size_t>(first + c), static_cast<std::size_t>(total_cells),
                mode == 0 ? ConditionMode::Ideal : ConditionMode::Realistic);
            const NewtonSystem sys = newton_system(mech, cond, ones, ones, h);
            std::memcpy(values + c * sys.a.nnz(), sys.a.values.data(),
                        sizeof(double) * sys.a.nnz());
            std::memcpy(rhs + c * species, sys.b.data(), sizeof(double) * species);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

typedef struct {
    int64_t step, newton_iterations, iterations_effective, iterations_sum;
    double max_residual_rms;
    int64_t wall_time_ns, breakdown_fallbacks, clip_events;
} ref_step_stats;

// run_simulation (simulate.cpp:72-178) on generate_mechanism(species,
// reactions, seed).  states: cells*species, in: initial, out: final.
// Returns -9 with *abort_step set on SolverAbort.
int ref_run_simulation(int64_t species, int64_t reactions, uint64_t seed, int64_t cells, int mode,
                       int64_t steps, double dt, double tol, int64_t max_iter, int strategy,
                       int64_t k_request, int direct, double newton_rtol, int64_t max_newton,
                       int64_t workers, double* states, ref_step_stats* stats, int64_t* abort_step) {
    if (abort_step) *abort_step = -1;
    try {
        const MechanismSpec mech = generate_mechanism(static_cast<std::size_t>(species),
                                                      static_cast<std::size_t>(reactions), seed);
        SimulationConfig cfg;
        cfg.cells = static_cast<std::size_t>(cells);
        cfg.mode = mode == 0 ? ConditionMode::Ideal : ConditionMode::Realistic;
        cfg.steps = static_cast<std::size_t>(steps);
        cfg.dt_seconds = dt;
        cfg.tol = tol;
        cfg.max_iter = static_cast<std::size_t>(max_iter);
        cfg.worker_count = static_cast<std::size_t>(workers);
        cfg.solver.use_direct_reference = direct != 0;
        cfg.solver.strategy.kind = strategy == 0 ? Strategy::OneCell
                                   : strategy == 1 ? Strategy::MultiCells
                                                   : Strategy::BlockCells;
        if (k_request > 0) cfg.solver.strategy.cells_per_block = static_cast<std::size_t>(k_request);
        cfg.newton_rtol = newton_rtol;
        cfg.max_newton_iterations = static_cast<std::size_t>(max_newton);
        std::vector<CellState> init(static_cast<std::size_t>(cells));
        for (int64_t c = 0; c < cells; ++c)
            init[c].concentrations.assign(states + c * species, states + (c + 1) * species);
        const SimulationResult r = run_simulation(mech, cfg, init);
        for (int64_t c = 0; c < cells; ++c)
            std::memcpy(states + c * species, r.final_states[c].concentrations.data(), sizeof(double) * species);
        for (std::size_t i = 0; i < r.per_step.size(); ++i) {
            const StepStats& q = r.per_step[i];
            stats[i] = ref_step_stats{static_cast<int64_t>(q.step), static_cast<int64_t>(q.newton_iterations),
                                      static_cast<int64_t>(q.iterations_effective),
                                      static_cast<int64_t>(q.iterations_sum), q.max_residual_rms,
                                      q.wall_time_ns, static_cast<int64_t>(q.breakdown_fallbacks),
                                      static_cast<int64_t>(q.clip_events)};
        }
        return 0;
    } catch (const SolverAbort& a) {
        if (abort_step) *abort_step = static_cast<int64_t>(a.step);
        return -9;
    } catch (...) {
        return map_exception();
    }
}

// format_double (format.cpp:9-14) into buf (>= 64 bytes).
int ref_format_double(double v, char* buf) {
    try {
        const std::string t = format_double(v);
        std::memcpy(buf, t.c_str(), t.size() + 1);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

namespace {
std::string g_text;  // last text result of the bench wrappers
}

// bench::to_csv (bench.cpp:189-218) of n rows given column-wise; strategy
// names are one NUL-separated block.  The text stays in ref_last_text().
int ref_to_csv(int64_t n, const int64_t* step, const char* strategies, const int64_t* cells,
               const int64_t* species, const double* cpb, const int64_t* it_eff, const int64_t* it_sum,
               const int64_t* wall, const double* rms, const int64_t* fallbacks, const int64_t* clips) {
    try {
        std::vector<bench::StepRecord> raw(static_cast<std::size_t>(n));
        const char* name = strategies;
        for (int64_t i = 0; i < n; ++i) {
            raw[i].step = static_cast<std::size_t>(step[i]);
            raw[i].strategy = name;
            name += raw[i].strategy.size() + 1;
            raw[i].cells = static_cast<std::size_t>(cells[i]);
            raw[i].species = static_cast<std::size_t>(species[i]);
            raw[i].cells_per_block = cpb[i];
            raw[i].iterations_effective = static_cast<std::size_t>(it_eff[i]);
            raw[i].iterations_sum = static_cast<std::size_t>(it_sum[i]);
            raw[i].wall_ns = wall[i];
            raw[i].max_residual_rms = rms[i];
            raw[i].breakdown_fallbacks = static_cast<std::size_t>(fallbacks[i]);
            raw[i].clip_events = static_cast<std::size_t>(clips[i]);
        }
        g_text = bench::to_csv(raw);
        if (bench::parse_csv(g_text) != raw) return -8;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// The reference reads a summary.json back (summary_stats_from_json,
// bench.cpp:332-357) and writes it again (summary_to_json) for the given
// config: strategies as kind (0/1/2) + k (0 = "N").  Text in ref_last_text().
int ref_summary_roundtrip(const char* json_in, int64_t cells, int64_t species, int64_t steps, double dt,
                          int mode, int64_t n_strat, const int32_t* kinds, const int64_t* ks, double tol,
                          int64_t max_iter, uint64_t seed, int64_t workers, const char* output_path) {
    try {
        bench::ExperimentConfig cfg;
        cfg.cells = static_cast<std::size_t>(cells);
        cfg.species = static_cast<std::size_t>(species);
        cfg.steps = static_cast<std::size_t>(steps);
        cfg.dt_seconds = dt;
        cfg.mode = mode == 0 ? ConditionMode::Ideal : ConditionMode::Realistic;
        for (int64_t i = 0; i < n_strat; ++i) {
            StrategyConfig sc;
            sc.kind = kinds[i] == 0 ? Strategy::OneCell : kinds[i] == 1 ? Strategy::MultiCells : Strategy::BlockCells;
            if (ks[i] > 0) sc.cells_per_block = static_cast<std::size_t>(ks[i]);
            cfg.strategies.push_back(sc);
        }
        cfg.tol = tol;
        cfg.max_iter = static_cast<std::size_t>(max_iter);
        cfg.seed = seed;
        cfg.worker_count = static_cast<std::size_t>(workers);
        cfg.output_path = output_path;
        const bench::AggregateStats stats = bench::summary_stats_from_json(json_in);
        g_text = bench::summary_to_json(cfg, stats);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// plan_kernel + occupancy_estimate + memory_estimate (exec_model.cpp:102-200)
// as the summary's JSON fragments, text in ref_last_text().
int ref_plan_json(int kind, int64_t cells, int64_t species, int64_t k, int64_t mtpb) {
    try {
        DeviceSpec dev;
        dev.max_threads_per_block = static_cast<std::size_t>(mtpb);
        if (dev.max_threads_per_sm < dev.max_threads_per_block) dev.max_threads_per_sm = dev.max_threads_per_block;
        const Strategy st = kind == 0 ? Strategy::OneCell : kind == 1 ? Strategy::MultiCells : Strategy::BlockCells;
        std::optional<std::size_t> req;
        if (k > 0) req = static_cast<std::size_t>(k);
        const KernelPlan plan = plan_kernel(st, static_cast<std::size_t>(cells), static_cast<std::size_t>(species),
                                            dev, st == Strategy::BlockCells ? req : std::nullopt);
        const OccupancyEstimate occ = occupancy_estimate(plan, dev);
        const auto opt = st == Strategy::BlockCells ? req : std::nullopt;
        g_text = kernel_plan_to_json(plan) + "\n" + format_double(occ.value) + " " +
                 (occ.shared_mem_exceeded ? "1" : "0") + " " +
                 std::to_string(memory_estimate(st, static_cast<std::size_t>(cells),
                                                static_cast<std::size_t>(species), 9, dev, opt)) +
                 " " +
                 std::to_string(memory_estimate(st, static_cast<std::size_t>(cells),
                                                static_cast<std::size_t>(species), BicgWorkspace::aux_array_count(),
                                                dev, opt));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

const char* ref_last_text() { return g_text.c_str(); }

}  // extern "C"
