// ref_bicgstab.cpp -- Jacobi-preconditioned BiCGSTAB composed from the
// UNMODIFIED reference's compiled primitives.  TEST INFRASTRUCTURE ONLY
// (linked into oracle/_ref/libbcref.so by oracle/Makefile; used by tests/ and
// bench.py's parity leg as the checker of the GPU BiCGSTAB path).
//
// The reference has no BiCGSTAB.  This file expresses the
// north-star algorithm with the reference's own code wherever an operation
// exists there, so that "pinned through the shared primitives" becomes
// "computed by the reference's primitives":
//   spmv             csr.cpp:90-101       (A y, A z, the fresh residual's A x)
//   axpby            csr.cpp:150-156      (every vector update, see below)
//   plan_reduce_map  reduction.hpp:60-79  (every dot product, its tree + host stage)
//   breakdown floor  bicg.cpp:10-14       (restated: file-local in bicg.cpp)
//   fresh residual   bicg.cpp:61-72       (restated with spmv + plan_reduce_map)
//   group solve      strategies.cpp:37-69 (assemble_block_diagonal, lu_solve fallback,
//                                          fallback residual through the same plan)
//   batch drivers    strategies.cpp:158-249 (plan_kernel, build_reduction_plan,
//                                          group partition, merge in group order)
// The only arithmetic not taken from the reference is the Jacobi scaling
// y_i = dinv_i * p_i (one correctly rounded multiply; the reference has no
// elementwise product) and dinv_i = 1.0 / a_ii.
//
// Vector updates as reference axpby calls (a*x + b*y: two products, one add):
//   p = r + beta*(p - omega*v)   ->  tmp = axpby(1, p, -omega, v); p = axpby(1, r, beta, tmp)
//     (1*p == p and (-omega)*v == -(omega*v) exactly, and p + (-(w)) == p - w,
//      so this is bit-identical to the restatement's p_i = r_i + beta*(p_i - omega*v_i))
//   s = r - alpha*v              ->  axpby(1, r, -alpha, v)
//   x = x + alpha*y              ->  axpby(1, x, alpha, y)
//   x = x + omega*z              ->  axpby(1, x, omega, z)
//   r = s - omega*t              ->  axpby(1, s, -omega, t)
// Semantics (x0, rho0 = alpha = omega = 1, the tt == 0 rule, breakdown order)
// are the ones oracle/bc_oracle.c documents (orc_bicgstab_solve) and DESIGN.md §3.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "blockcells/bicg.hpp"
#include "blockcells/csr.hpp"
#include "blockcells/dense_lu.hpp"
#include "blockcells/exec_model.hpp"
#include "blockcells/reduction.hpp"
#include "blockcells/strategies.hpp"

using namespace blockcells;

namespace {

constexpr double kFloor = 1e-300;  // bicg.cpp:10
bool breaks(double v) { return !std::isfinite(v) || std::abs(v) < kFloor; }  // bicg.cpp:12-14

struct StabWs {
    DenseVector r, rh, p, v, y, s, z, t, dinv, ax, tmp;
    std::vector<double> scratch;
};

SolveOutcome bicgstab_solve_ref(const CsrMatrix& a, const DenseVector& b, const DenseVector& x0,
                                double tol, std::size_t max_iter, const ReductionPlan& plan,
                                StabWs& ws) {
    if (a.n_rows != a.n_cols) throw std::invalid_argument("bicgstab: matrix not square");
    const std::size_t n = a.n_rows;
    if (b.size() != n || x0.size() != n) throw std::invalid_argument("bicgstab: dimension mismatch");
    if (!(tol > 0.0)) throw std::invalid_argument("bicgstab: tol must be positive");
    if (max_iter < 1) throw std::invalid_argument("bicgstab: max_iter must be >= 1");
    plan.check_partition(n);

    auto dot = [&](const DenseVector& u, const DenseVector& w) {
        return plan_reduce_map(n, [&](std::size_t i) { return u[i] * w[i]; }, plan, ws.scratch);
    };
    auto residual_rms = [&](const DenseVector& x) {  // bicg.cpp:61-72
        spmv(a, x, ws.ax);
        const double sq = plan_reduce_map(
            n,
            [&](std::size_t i) {
                const double ri = b[i] - ws.ax[i];
                return ri * ri;
            },
            plan, ws.scratch);
        return std::sqrt(sq / static_cast<double>(n));
    };

    SolveOutcome out;
    out.x = x0;
    ws.dinv.assign(n, 1.0);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = a.row_ptr[i]; j < a.row_ptr[i + 1]; ++j)
            if (a.col_idx[j] == i) {
                if (a.values[j] != 0.0) ws.dinv[i] = 1.0 / a.values[j];
                break;
            }

    spmv(a, out.x, ws.ax);
    axpby(1.0, b, -1.0, ws.ax, ws.r);
    ws.rh = ws.r;
    ws.p.assign(n, 0.0);
    ws.v.assign(n, 0.0);
    ws.y.resize(n);
    ws.z.resize(n);

    double sigma = dot(ws.r, ws.r);
    if (std::sqrt(sigma / static_cast<double>(n)) <= tol) {
        out.final_residual_rms = residual_rms(out.x);
        out.converged = out.final_residual_rms <= tol;
        if (out.converged) return out;
    }

    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    for (std::size_t iter = 1; iter <= max_iter; ++iter) {
        const double rho = dot(ws.rh, ws.r);
        if (breaks(rho)) { out.breakdown = true; break; }
        const double beta = (rho / rho_prev) * (alpha / omega);
        axpby(1.0, ws.p, -omega, ws.v, ws.tmp);
        axpby(1.0, ws.r, beta, ws.tmp, ws.p);
        for (std::size_t i = 0; i < n; ++i) ws.y[i] = ws.dinv[i] * ws.p[i];
        spmv(a, ws.y, ws.v);
        const double den = dot(ws.rh, ws.v);
        if (breaks(den)) { out.breakdown = true; break; }
        alpha = rho / den;
        axpby(1.0, ws.r, -alpha, ws.v, ws.s);
        for (std::size_t i = 0; i < n; ++i) ws.z[i] = ws.dinv[i] * ws.s[i];
        axpby(1.0, out.x, alpha, ws.y, out.x);
        spmv(a, ws.z, ws.t);
        const double tt = dot(ws.t, ws.t);
        const double ts = dot(ws.t, ws.s);
        if (tt != 0.0 && breaks(tt)) { out.breakdown = true; break; }
        omega = tt == 0.0 ? 0.0 : ts / tt;
        axpby(1.0, out.x, omega, ws.z, out.x);
        axpby(1.0, ws.s, -omega, ws.t, ws.r);
        rho_prev = rho;
        out.iterations = iter;

        sigma = dot(ws.r, ws.r);
        if (!std::isfinite(sigma)) { out.breakdown = true; break; }
        if (std::sqrt(sigma / static_cast<double>(n)) <= tol) {
            const double fresh = residual_rms(out.x);
            if (fresh <= tol) {
                out.final_residual_rms = fresh;
                out.converged = true;
                return out;
            }
        }
        if (breaks(omega)) { out.breakdown = true; break; }
    }
    out.final_residual_rms = residual_rms(out.x);
    out.converged = !out.breakdown && out.final_residual_rms <= tol;
    return out;
}

struct GroupOut {
    std::size_t iterations = 0;
    double rms = 0.0;
    bool fell_back = false, converged = false, breakdown = false;
};

// strategies.cpp:37-69 solve_group with the composed BiCGSTAB; x written in place.
GroupOut solve_group_stab(const BatchedSystem& sys, IndexRange cells, const ReductionPlan& plan,
                          double tol, std::size_t max_iter, StabWs& ws, double* x_out) {
    const auto [a, b] = assemble_block_diagonal(sys, cells);
    SolveOutcome o = bicgstab_solve_ref(a, b, DenseVector(b.size(), 0.0), tol, max_iter, plan, ws);
    GroupOut g;
    g.iterations = o.iterations;
    g.converged = o.converged;
    g.breakdown = o.breakdown;
    if (o.breakdown) {
        o.x = lu_solve(a, b);
        g.fell_back = true;
        const DenseVector ax = spmv(a, o.x);
        std::vector<double> scratch;
        const double sq = plan_reduce_map(
            b.size(),
            [&](std::size_t i) {
                const double ri = b[i] - ax[i];
                return ri * ri;
            },
            plan, scratch);
        o.final_residual_rms = std::sqrt(sq / static_cast<double>(b.size()));
    }
    g.rms = o.final_residual_rms;
    std::memcpy(x_out + cells.begin * sys.species, o.x.data(), sizeof(double) * o.x.size());
    return g;
}

int map_exc() {
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

}  // namespace

extern "C" {

// Single system, explicit plan (ranges as pairs), as ref_bicg_solve.
int ref_bicgstab_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                       const double* b, const double* x0, double tol, int64_t max_iter,
                       const int64_t* ranges, int64_t n_blocks, int host_stage, double* x_out,
                       int64_t* iterations, double* rms, int32_t* converged, int32_t* breakdown) {
    try {
        CsrMatrix a;
        a.n_rows = a.n_cols = static_cast<std::size_t>(n);
        a.row_ptr.assign(rp, rp + n + 1);
        a.col_idx.assign(ci, ci + rp[n]);
        a.values.assign(va, va + rp[n]);
        ReductionPlan plan;
        for (int64_t k = 0; k < n_blocks; ++k)
            plan.block_ranges.push_back({static_cast<std::size_t>(ranges[2 * k]),
                                         static_cast<std::size_t>(ranges[2 * k + 1])});
        plan.host_stage = host_stage != 0;
        StabWs ws;
        const SolveOutcome o = bicgstab_solve_ref(a, DenseVector(b, b + n), DenseVector(x0, x0 + n), tol,
                                                  static_cast<std::size_t>(max_iter), plan, ws);
        std::memcpy(x_out, o.x.data(), sizeof(double) * n);
        *iterations = static_cast<int64_t>(o.iterations);
        *rms = o.final_residual_rms;
        *converged = o.converged;
        *breakdown = o.breakdown;
        return 0;
    } catch (...) {
        return map_exc();
    }
}

typedef struct {
    int64_t n_groups, iterations_effective, iterations_sum;
    double max_residual_rms;
    int64_t breakdown_fallbacks;
    double cells_per_block;
    int64_t wall_time_ns;
} ref_stab_report;

}  // extern "C"

namespace {

BatchedSystem* make_system(int64_t species, int64_t cells, const int32_t* row_ptr, const int32_t* col_idx,
                           const double* values, const double* rhs) {
    auto* sys = new BatchedSystem();
    sys->species = static_cast<std::size_t>(species);
    sys->cells = static_cast<std::size_t>(cells);
    const int64_t nnz = row_ptr[species];
    CsrMatrix proto;
    proto.n_rows = proto.n_cols = sys->species;
    proto.row_ptr.assign(row_ptr, row_ptr + species + 1);
    proto.col_idx.assign(col_idx, col_idx + nnz);
    sys->per_cell_matrices.reserve(sys->cells);
    sys->per_cell_rhs.reserve(sys->cells);
    for (int64_t c = 0; c < cells; ++c) {
        CsrMatrix m = proto;
        m.values.assign(values + c * nnz, values + (c + 1) * nnz);
        sys->per_cell_matrices.push_back(std::move(m));
        sys->per_cell_rhs.emplace_back(rhs + c * species, rhs + (c + 1) * species);
    }
    return sys;
}

Strategy kind_of(int strategy) {
    return strategy == 0 ? Strategy::OneCell : strategy == 1 ? Strategy::MultiCells : Strategy::BlockCells;
}

DeviceSpec device_of(int64_t max_threads_per_block) {
    DeviceSpec dev;
    dev.max_threads_per_block = static_cast<std::size_t>(max_threads_per_block);
    if (dev.max_threads_per_sm < dev.max_threads_per_block) dev.max_threads_per_sm = dev.max_threads_per_block;
    return dev;
}

// run_strategy's drivers (strategies.cpp:158-249) with the composed BiCGSTAB
// as the group solver.  wall_time_ns covers the same span as the
// reference's SolveReport::wall_time_ns (check() excluded, as there it
// precedes the clock start).
void solve_batch_stab(const BatchedSystem& sys, int strategy, int64_t k_request, double tol, int64_t max_iter,
                      int64_t max_threads_per_block, int64_t workers, double* x_out, int64_t* group_iters,
                      double* group_rms, uint8_t* group_flags, ref_stab_report* report) {
    sys.check();
    const auto start = std::chrono::steady_clock::now();
    const DeviceSpec dev = device_of(max_threads_per_block);
    const Strategy kind = kind_of(strategy);
    std::optional<std::size_t> req;
    if (strategy == 2 && k_request > 0) req = static_cast<std::size_t>(k_request);
    const KernelPlan kp = plan_kernel(kind, sys.cells, sys.species, dev, req);

    std::vector<IndexRange> ranges;
    ReductionPlan full, rem;
    std::size_t k = 1;
    if (kind == Strategy::MultiCells) {
        ranges.push_back({0, sys.cells});
        full = build_reduction_plan(kp, sys.cells * sys.species);  // strategies.cpp:182-184
    } else if (kind == Strategy::OneCell) {
        for (std::size_t c = 0; c < sys.cells; ++c) ranges.push_back({c, c + 1});
        full = build_reduction_plan(kp, sys.species);  // strategies.cpp:163-164
    } else {
        k = static_cast<std::size_t>(kp.cells_per_block);
        if (k == 0) throw InvalidGrouping("block-cells: species exceed the block size");
        for (std::size_t c = 0; c + k <= sys.cells; c += k) ranges.push_back({c, c + k});
        if (const std::size_t left = sys.cells % k; left != 0) ranges.push_back({sys.cells - left, sys.cells});
        full = build_reduction_plan(kp, k * sys.species);  // strategies.cpp:215-219
        if (kp.remainder) rem = ReductionPlan::single_block(kp.remainder->threads);
    }
    std::vector<GroupOut> out(ranges.size());
    std::size_t nw = kind == Strategy::BlockCells ? static_cast<std::size_t>(workers) : 1;
    if (nw == 0) nw = std::max(1u, std::thread::hardware_concurrency());
    nw = std::max<std::size_t>(1, std::min(nw, ranges.size()));
    std::atomic<std::size_t> next{0};
    auto work = [&] {
        StabWs ws;
        for (;;) {
            const std::size_t g = next.fetch_add(1);
            if (g >= ranges.size()) return;
            const ReductionPlan& plan = (kind == Strategy::BlockCells && ranges[g].size() != k) ? rem : full;
            out[g] = solve_group_stab(sys, ranges[g], plan, tol, static_cast<std::size_t>(max_iter), ws, x_out);
        }
    };
    if (nw <= 1) {
        work();
    } else {
        std::vector<std::thread> pool;
        for (std::size_t w = 0; w < nw; ++w) pool.emplace_back(work);
        for (auto& t : pool) t.join();
    }
    // merge_groups (strategies.cpp:71-87)
    ref_stab_report r{};
    r.n_groups = static_cast<int64_t>(out.size());
    r.cells_per_block = kp.cells_per_block;
    for (std::size_t g = 0; g < out.size(); ++g) {
        const GroupOut& o = out[g];
        r.iterations_sum += static_cast<int64_t>(o.iterations);
        r.iterations_effective = std::max<int64_t>(r.iterations_effective, static_cast<int64_t>(o.iterations));
        r.max_residual_rms = std::max(r.max_residual_rms, o.rms);
        r.breakdown_fallbacks += o.fell_back ? 1 : 0;
        if (group_iters) group_iters[g] = static_cast<int64_t>(o.iterations);
        if (group_rms) group_rms[g] = o.rms;
        if (group_flags) group_flags[g] = static_cast<uint8_t>((o.converged ? 1 : 0) | (o.breakdown ? 2 : 0) |
                                                               (o.fell_back ? 4 : 0));
    }
    r.wall_time_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                         std::chrono::steady_clock::now() - start).count();
    if (report) *report = r;
}

}  // namespace

extern "C" {

// One-shot: build the BatchedSystem, solve, free.  strategy: 0 one-cell,
// 1 multi-cells, 2 block-cells (k_request 0 = "N").  Per-group outputs in
// group order: iterations, final rms, flags (bit 0 converged, bit 1
// breakdown, bit 2 LU fallback: ORC_FLAG_*).
int ref_solve_batch_bicgstab(int strategy, int64_t k_request, int64_t species, int64_t cells,
                             const int32_t* row_ptr, const int32_t* col_idx, const double* values,
                             const double* rhs, double tol, int64_t max_iter,
                             int64_t max_threads_per_block, int64_t workers, double* x_out,
                             int64_t* group_iters, double* group_rms, uint8_t* group_flags,
                             ref_stab_report* report) {
    BatchedSystem* sys = nullptr;
    try {
        sys = make_system(species, cells, row_ptr, col_idx, values, rhs);
        solve_batch_stab(*sys, strategy, k_request, tol, max_iter, max_threads_per_block, workers, x_out,
                         group_iters, group_rms, group_flags, report);
        delete sys;
        return 0;
    } catch (...) {
        delete sys;
        return map_exc();
    }
}

// A resident BatchedSystem (the reference's host form, strategies.hpp:15-23)
// for repeated timed solves: bench.py's reference arm builds it once, so a
// timed step is exactly the reference's run_strategy call.
void* ref_batch_create(int64_t species, int64_t cells, const int32_t* row_ptr, const int32_t* col_idx,
                       const double* values, const double* rhs) {
    try {
        return make_system(species, cells, row_ptr, col_idx, values, rhs);
    } catch (...) {
        return nullptr;
    }
}

void ref_batch_destroy(void* h) { delete static_cast<BatchedSystem*>(h); }

// algo 0: the reference's stock run_strategy (strategies.cpp:251-264, BiCG;
// group rms/flags are not in its SolveReport and stay untouched);
// algo 1: the composed Jacobi-BiCGSTAB through the same drivers.
int ref_batch_run(void* h, int algo, int strategy, int64_t k_request, double tol, int64_t max_iter,
                  int64_t max_threads_per_block, int64_t workers, double* x_out, int64_t* group_iters,
                  double* group_rms, uint8_t* group_flags, ref_stab_report* report) {
    try {
        const BatchedSystem& sys = *static_cast<const BatchedSystem*>(h);
        if (algo == 1) {
            solve_batch_stab(sys, strategy, k_request, tol, max_iter, max_threads_per_block, workers, x_out,
                             group_iters, group_rms, group_flags, report);
            return 0;
        }
        StrategyConfig cfg;
        cfg.kind = kind_of(strategy);
        if (strategy == 2 && k_request > 0) cfg.cells_per_block = static_cast<std::size_t>(k_request);
        const SolveReport rep = run_strategy(sys, cfg, device_of(max_threads_per_block), tol,
                                             static_cast<std::size_t>(max_iter), static_cast<std::size_t>(workers));
        for (std::size_t c = 0; c < sys.cells; ++c)
            std::memcpy(x_out + c * sys.species, rep.per_cell_x[c].data(), sizeof(double) * sys.species);
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
        return map_exc();
    }
}

}  // extern "C"
