// blockcells_b200_shim.cpp -- drop-in replacement for the reference's
// proj/core/src/strategies.cpp and proj/core/src/bicg.cpp.
//
// It defines every symbol those two files define, with the same signatures
// (strategies.hpp:15-90, bicg.hpp:11-53), and routes the solves through the
// C ABI of libbc_b200.so (include/blockcells_b200.h), i.e. through the fused
// sm_100a kernels.  Built against the reference's public headers; linked with
// the rest of the reference library (csr/reduction/exec_model/dense_lu/...)
// in place of the two replaced files.  See INTEGRATION.md.
//
// Semantics kept from the reference:
//   * argument checks and exception types (BatchedSystem::check, plan_kernel's
//     InvalidGrouping / UnsupportedMechanism, bicg's invalid_argument,
//     SingularMatrix from the LU fallback);
//   * results: per_cell_x, per_block_iterations, iterations_effective/sum,
//     max_residual_rms, breakdown_fallbacks, cells_per_block -- bit-identical to
//     the reference for the default algorithm (BiCG);
//   * wall_time_ns covers the whole call (strategies.cpp:15-21).
// worker_count is accepted and ignored: the GPU result does not depend on it,
// as the reference's does not (tests/test_strategies.cpp:254-268).
//
// Additions (blockcells_b200_shim.hpp): the Jacobi-BiCGSTAB algorithm
// selector and bicgstab_solve with bicg_solve's shape.
#include "blockcells_b200_shim.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "blockcells/dense_lu.hpp"
#include "blockcells_b200.h"
#include "blockcells_workload.h"

namespace blockcells {

namespace {

using Clock = std::chrono::steady_clock;

std::int64_t elapsed_ns(Clock::time_point start) {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - start).count();
}

thread_local b200::Algorithm t_algorithm = b200::Algorithm::BiCG;

b200::Algorithm env_algorithm() {
    const char* e = std::getenv("BLOCKCELLS_B200_ALGO");
    if (e && std::string(e) == "bicgstab") return b200::Algorithm::JacobiBiCGStab;
    return t_algorithm;
}

// One context per (calling thread, device): contexts are not thread-safe.
struct CtxHolder {
    bc_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) bc_ctx_destroy(ctx);
    }
};

bc_ctx* context() {
    thread_local CtxHolder h;
    if (!h.ctx) {
        int dev = 0;
        if (const char* e = std::getenv("BLOCKCELLS_B200_DEVICE")) dev = std::atoi(e);
        const int st = bc_ctx_create(dev, &h.ctx);
        if (st != BC_OK) throw std::runtime_error("blockcells_b200: no usable sm_100a device (status " +
                                                  std::to_string(st) + ")");
    }
    return h.ctx;
}

// BLOCKCELLS_B200_DEVICES="0,1,...,7": the batched strategies run on a
// device set (bc_devset_solve: contiguous group-aligned shards, one host
// thread per GPU, merge in group order -- SURVEY.md §8e), so the reference's
// own callers (run_simulation -> run_strategy, simulate.cpp:137-140) use every
// listed GPU with no change.  Unset: one device (BLOCKCELLS_B200_DEVICE).
struct SetHolder {
    bc_devset* set = nullptr;
    bool probed = false;
    ~SetHolder() {
        if (set) bc_devset_destroy(set);
    }
};

bc_devset* device_set() {
    thread_local SetHolder h;
    if (!h.probed) {
        h.probed = true;
        const char* e = std::getenv("BLOCKCELLS_B200_DEVICES");
        if (!e || !*e) return nullptr;
        std::vector<int> devs;
        std::string spec(e);
        for (std::size_t pos = 0; pos <= spec.size();) {
            const std::size_t next = std::min(spec.find(',', pos), spec.size());
            if (next > pos) devs.push_back(std::atoi(spec.substr(pos, next - pos).c_str()));
            pos = next + 1;
        }
        if (devs.empty()) return nullptr;
        const int st = bc_devset_create(static_cast<int>(devs.size()), devs.data(), &h.set);
        if (st != BC_OK)
            throw std::runtime_error("blockcells_b200: cannot open the devices in BLOCKCELLS_B200_DEVICES (status " +
                                     std::to_string(st) + ")");
    }
    return h.set;
}

// Pinned staging for the C ABI's flat arrays, reused across calls (grown on
// demand): pinned inputs stream into the solve while it runs and the kernels
// write x into pinned memory in place.
struct Staging {
    void* p = nullptr;
    std::size_t bytes = 0;
    ~Staging() { bc_host_free(p); }
    double* get(std::size_t want) {
        if (want > bytes) {
            bc_host_free(p);
            p = nullptr;
            bytes = 0;
            if (bc_host_alloc(want, &p) != BC_OK) throw std::bad_alloc();
            bytes = want;
        }
        return static_cast<double*>(p);
    }
};

// Host threads for packing / unpacking / checking (the results do not depend
// on them, as the reference's do not depend on worker_count).
std::size_t host_threads(std::size_t worker_count) {
    const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
    return worker_count == 0 ? hw : std::max(worker_count, std::min<std::size_t>(hw, 8));
}

template <class F>
void parallel_for(std::size_t n, std::size_t threads, F&& f) {
    threads = std::max<std::size_t>(1, std::min(threads, n / 256 + 1));
    if (threads == 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t < threads; ++t)
        pool.emplace_back([&, t] { f(n * t / threads, n * (t + 1) / threads); });
    for (std::thread& th : pool) th.join();
}

[[noreturn]] void raise_status(int st, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (st) {
        case BC_ERR_INVALID_GROUPING: throw InvalidGrouping(m);
        case BC_ERR_UNSUPPORTED_MECHANISM: throw UnsupportedMechanism(m);
        case BC_ERR_SINGULAR_MATRIX: throw SingularMatrix(m);
        case BC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case BC_ERR_NO_MEMORY: throw std::bad_alloc();
        default: throw std::runtime_error("blockcells_b200: " + m);
    }
}

void check(bc_ctx* ctx, int st) {
    if (st != BC_OK) raise_status(st, bc_last_error(ctx));
}

// BatchedSystem::check (strategies.cpp:91-107) over host threads: each
// thread finds the first bad cell of its range; the lowest one is reported,
// so the exception is the one the sequential loop throws.
void check_system(const BatchedSystem& system, std::size_t threads) {
    if (system.cells == 0) throw std::invalid_argument("batched system: no cells");
    if (system.species == 0) throw std::invalid_argument("batched system: no species");
    if (system.per_cell_matrices.size() != system.cells || system.per_cell_rhs.size() != system.cells)
        throw std::invalid_argument("batched system: per-cell arrays mismatch");
    const CsrMatrix& first = system.per_cell_matrices.front();
    const std::size_t n = system.cells, none = n;
    const std::size_t nt = std::max<std::size_t>(1, std::min(threads, n / 256 + 1));
    std::vector<std::size_t> bad_m(nt, none), bad_b(nt, none);
    std::vector<int> why(nt, 0);
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (std::size_t c = n * t / nt; c < n * (t + 1) / nt; ++c) {
                const CsrMatrix& m = system.per_cell_matrices[c];
                if (m.n_rows != system.species || m.n_cols != system.species) {
                    bad_m[t] = c, why[t] = 1;
                    break;
                }
                if (m.row_ptr != first.row_ptr || m.col_idx != first.col_idx) {
                    bad_m[t] = c, why[t] = 2;
                    break;
                }
            }
            for (std::size_t c = n * t / nt; c < n * (t + 1) / nt; ++c)
                if (system.per_cell_rhs[c].size() != system.species) {
                    bad_b[t] = c;
                    break;
                }
        });
    for (std::thread& th : pool) th.join();
    for (std::size_t t = 0; t < nt; ++t)
        if (bad_m[t] != none)
            throw std::invalid_argument(why[t] == 1 ? "batched system: cell matrix dimension"
                                                    : "batched system: cells do not share one sparsity pattern");
    for (std::size_t t = 0; t < nt; ++t)
        if (bad_b[t] != none) throw std::invalid_argument("batched system: rhs dimension");
}

// Everything BatchedSystem::check tests except the per-cell pattern
// comparison (the 1.7k-index compare per cell that dominates it): true when
// it all holds.  Then the only error check() can still throw is the pattern
// mismatch of the lowest such cell, which run_gpu tests piece by piece
// (pack_checked) before each piece is handed to the GPU.
bool light_check(const BatchedSystem& system, std::size_t threads) {
    if (system.cells == 0 || system.species == 0 || system.per_cell_matrices.size() != system.cells ||
        system.per_cell_rhs.size() != system.cells)
        return false;
    const std::size_t n = system.cells;
    std::vector<char> ok(std::max<std::size_t>(1, std::min(threads, n / 256 + 1)), 1);
    const std::size_t nt = ok.size();
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (std::size_t c = n * t / nt; c < n * (t + 1) / nt && ok[t]; ++c) {
                const CsrMatrix& m = system.per_cell_matrices[c];
                ok[t] = m.n_rows == system.species && m.n_cols == system.species &&
                        system.per_cell_rhs[c].size() == system.species;
            }
        });
    for (std::thread& th : pool) th.join();
    return std::all_of(ok.begin(), ok.end(), [](char v) { return v != 0; });
}

SolveReport run_gpu(const BatchedSystem& system, int strategy, std::optional<std::size_t> k,
                    const DeviceSpec& device, double tol, std::size_t max_iter, Strategy kind,
                    std::size_t worker_count = 1) {
    const std::size_t threads = host_threads(worker_count);
    // strategies.cpp:91-107: anything but a pattern mismatch is found here and
    // thrown exactly as check() does; pattern mismatches below, before the
    // cells concerned are solved, lowest cell first
    if (!light_check(system, threads)) check_system(system, threads);
    const auto start = Clock::now();
    bc_devset* set = device_set();
    bc_ctx* ctx = set ? nullptr : context();
    const CsrMatrix& first = system.per_cell_matrices.front();
    {
        const std::vector<int32_t> rp(first.row_ptr.begin(), first.row_ptr.end()),
            ci(first.col_idx.begin(), first.col_idx.end());
        const int st = set ? bc_devset_set_pattern(set, static_cast<int32_t>(system.species), rp.data(), ci.data())
                           : bc_set_pattern(ctx, static_cast<int32_t>(system.species), rp.data(), ci.data());
        if (st != BC_OK) raise_status(st, set ? bc_devset_last_error(set) : bc_last_error(ctx));
    }
    const std::size_t s = system.species, cells = system.cells, nnz = first.nnz();
    bc_solve_params prm{};
    prm.strategy = strategy;
    prm.algo = env_algorithm() == b200::Algorithm::BiCG ? BC_ALGO_BICG : BC_ALGO_BICGSTAB_JACOBI;
    if (k) {
        if (*k < 1) throw std::invalid_argument("plan_kernel: cells per block must be >= 1");
        prm.cells_per_block = static_cast<int64_t>(*k);
    }
    prm.cells = static_cast<int64_t>(cells);
    prm.tol = tol;
    prm.max_iter = static_cast<int64_t>(std::min<std::size_t>(max_iter, INT64_MAX));
    prm.max_threads_per_block = static_cast<int64_t>(device.max_threads_per_block);
    device.check();
    int64_t n_groups = 0;
    double cpb = 0;
    {
        const int st = bc_plan(static_cast<int32_t>(s), &prm, &n_groups, &cpb);
        if (st != BC_OK) raise_status(st, set ? bc_devset_last_error(set) : bc_last_error(ctx));
    }
    // pack BatchedSystem -> the C ABI's cell-major arrays, in pinned staging
    thread_local Staging st_values, st_rhs, st_x;
    double* values = st_values.get(sizeof(double) * cells * nnz);
    double* rhs = st_rhs.get(sizeof(double) * cells * s);
    double* x = st_x.get(sizeof(double) * cells * s);
    std::vector<int32_t> iters(n_groups);
    SolveReport report;  // merge_groups, strategies.cpp:71-87
    report.strategy = kind;
    report.per_cell_x.resize(cells);
    // pattern check (check()'s remaining test) and pack, one pass per cell;
    // throws check()'s error for the lowest mismatching cell of [a, b)
    auto pack = [&](std::size_t a, std::size_t b) {
        const std::size_t none = b;
        std::mutex bad_mu;
        std::size_t bad = none;
        parallel_for(b - a, threads, [&](std::size_t c0, std::size_t c1) {
            for (std::size_t c = a + c0; c < a + c1; ++c) {
                const CsrMatrix& m = system.per_cell_matrices[c];
                if (c > 0 && (m.row_ptr != first.row_ptr || m.col_idx != first.col_idx)) {
                    std::lock_guard<std::mutex> lk(bad_mu);
                    bad = std::min(bad, c);
                    return;
                }
                std::memcpy(values + c * nnz, m.values.data(), sizeof(double) * nnz);
                std::memcpy(rhs + c * s, system.per_cell_rhs[c].data(), sizeof(double) * s);
            }
        });
        if (bad != none) throw std::invalid_argument("batched system: cells do not share one sparsity pattern");
    };
    auto unpack = [&](std::size_t a, std::size_t b) {
        parallel_for(b - a, threads, [&](std::size_t c0, std::size_t c1) {
            for (std::size_t c = a + c0; c < a + c1; ++c) report.per_cell_x[c].assign(x + c * s, x + (c + 1) * s);
        });
    };
    // Independent groups (One-cell, Block-cells(k), thread-per-cell) on one
    // device: the batch in kPieces group-aligned pieces, each solved on the GPU
    // (a solver thread) while the host packs the next and unpacks the previous,
    // so packing and unpacking leave the critical path.  Each piece is its own
    // bc_solve over disjoint groups, folded below as merge_groups folds groups:
    // outputs bit-identical to one call.  BLOCKCELLS_B200_OVERLAP=0: one call.
    int kPieces = 4;
    if (const char* e = std::getenv("BLOCKCELLS_B200_PIECES")) kPieces = std::max(2, std::min(64, std::atoi(e)));
    // the first piece, whose packing nothing overlaps, as a fraction of the
    // batch in 1/64ths; the rest in equal shares.  B200, 100k M156 cells:
    // 4 pieces with a 1/16 first piece 538k cell-solves/s, equal quarters
    // 526k, 3 pieces 532k, 6 pieces 538k, 8 pieces 493-525k, 2 pieces 508k
    int first64 = 4;
    if (const char* e = std::getenv("BLOCKCELLS_B200_FIRST64")) first64 = std::max(1, std::min(63, std::atoi(e)));
    constexpr std::size_t kOverlapMinCells = 16384;
    const char* ov = std::getenv("BLOCKCELLS_B200_OVERLAP");
    const bool independent = strategy == BC_STRATEGY_BLOCK_CELLS || strategy == BC_STRATEGY_ONE_CELL ||
                             strategy == BC_STRATEGY_THREAD_PER_CELL;
    const std::size_t kg = strategy == BC_STRATEGY_BLOCK_CELLS ? static_cast<std::size_t>(cpb) : 1;
    const int pieces = (!set && independent && kg >= 1 && cells >= kOverlapMinCells && !(ov && *ov == '0'))
                           ? kPieces : 1;
    std::vector<std::size_t> cut(pieces + 1, cells);
    for (int b = 0; b < pieces; ++b) {
        const std::size_t c0 = cells * first64 / 64;  // then equal shares of the rest
        cut[b] = (b == 0 ? 0 : c0 + (cells - c0) * (b - 1) / (pieces - 1)) / kg * kg;
    }
    std::vector<bc_report> reps(pieces);
    if (pieces == 1) {
        pack(0, cells);
        const int st = set ? bc_devset_solve(set, &prm, values, rhs, x, iters.data(), nullptr, nullptr, &reps[0])
                           : bc_solve(ctx, &prm, values, rhs, x, iters.data(), nullptr, nullptr, &reps[0]);
        if (st != BC_OK) raise_status(st, set ? bc_devset_last_error(set) : bc_last_error(ctx));
        unpack(0, cells);
    } else {
        std::mutex mu;
        std::condition_variable cv;
        int packed = 0, solved = 0, status = BC_OK;
        bool cancel = false;  // the host side threw: the solver thread stops
        std::string err;
        std::thread solver([&] {
            for (int b = 0; b < pieces; ++b) {
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return packed > b || cancel; });
                    if (cancel) return;
                }
                int st = BC_OK;
                if (cut[b + 1] > cut[b]) {
                    bc_solve_params sub = prm;
                    sub.cells = static_cast<int64_t>(cut[b + 1] - cut[b]);
                    st = bc_solve(ctx, &sub, values + cut[b] * nnz, rhs + cut[b] * s, x + cut[b] * s,
                                  iters.data() + cut[b] / kg, nullptr, nullptr, &reps[b]);
                }
                std::lock_guard<std::mutex> lk(mu);
                if (st != BC_OK) {
                    status = st;
                    err = bc_last_error(ctx);
                    solved = pieces;  // the main thread stops waiting
                } else {
                    solved = b + 1;
                }
                cv.notify_all();
                if (st != BC_OK) return;
            }
        });
        try {
            for (int b = 0; b < pieces; ++b) {
                pack(cut[b], cut[b + 1]);
                std::lock_guard<std::mutex> lk(mu);
                packed = b + 1;
                cv.notify_all();
            }
            for (int b = 0; b < pieces; ++b) {
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return solved > b; });
                    if (status != BC_OK) break;
                }
                unpack(cut[b], cut[b + 1]);
            }
        } catch (...) {
            {
                std::lock_guard<std::mutex> lk(mu);
                cancel = true;
                cv.notify_all();
            }
            solver.join();
            throw;
        }
        solver.join();
        if (status != BC_OK) raise_status(status, err.c_str());
    }
    bc_report rep{};  // the pieces folded in group order (bc_devset_solve's merge)
    rep.cells_per_block = cpb;
    for (int b = 0; b < pieces; ++b) {
        if (cut[b + 1] == cut[b] && pieces > 1) continue;
        const bc_report& q = reps[b];
        rep.iterations_sum += q.iterations_sum;
        rep.iterations_effective = std::max(rep.iterations_effective, q.iterations_effective);
        rep.max_residual_rms = std::max(rep.max_residual_rms, q.max_residual_rms);
        rep.breakdown_fallbacks += q.breakdown_fallbacks;
        if (pieces == 1) rep.cells_per_block = q.cells_per_block;
    }
    report.cells_per_block = rep.cells_per_block;
    report.per_block_iterations.assign(iters.begin(), iters.end());
    report.iterations_sum = static_cast<std::size_t>(rep.iterations_sum);
    report.iterations_effective = static_cast<std::size_t>(rep.iterations_effective);
    report.max_residual_rms = rep.max_residual_rms;
    report.breakdown_fallbacks = static_cast<std::size_t>(rep.breakdown_fallbacks);
    report.wall_time_ns = elapsed_ns(start);
    return report;
}

SolveOutcome single_system(b200::Algorithm algo, const CsrMatrix& a, const DenseVector& b, const DenseVector& x0,
                           double tol, std::size_t max_iter, const ReductionPlan& reduction) {
    if (a.n_rows != a.n_cols) throw std::invalid_argument("bicg: matrix not square");
    const std::size_t n = a.n_rows;
    if (b.size() != n || x0.size() != n) throw std::invalid_argument("bicg: dimension mismatch");
    if (!(tol > 0.0)) throw std::invalid_argument("bicg: tol must be positive");
    if (max_iter < 1) throw std::invalid_argument("bicg: max_iter must be >= 1");
    reduction.check_partition(n);
    bc_ctx* ctx = context();
    std::vector<int32_t> rp(a.row_ptr.begin(), a.row_ptr.end()), ci(a.col_idx.begin(), a.col_idx.end());
    std::vector<int64_t> ranges;
    for (const IndexRange& r : reduction.block_ranges) {
        ranges.push_back(static_cast<int64_t>(r.begin));
        ranges.push_back(static_cast<int64_t>(r.end));
    }
    SolveOutcome out;
    out.x.resize(n);
    bc_outcome o{};
    check(ctx, bc_bicg_solve(ctx, algo == b200::Algorithm::BiCG ? BC_ALGO_BICG : BC_ALGO_BICGSTAB_JACOBI,
                             static_cast<int32_t>(n), rp.data(), ci.data(), a.values.data(), b.data(), x0.data(), tol,
                             static_cast<int64_t>(max_iter), static_cast<int64_t>(reduction.n_blocks()),
                             ranges.data(), out.x.data(), &o));
    out.iterations = static_cast<std::size_t>(o.iterations);
    out.final_residual_rms = o.final_residual_rms;
    out.converged = o.converged != 0;
    out.breakdown = o.breakdown != 0;
    return out;
}

}  // namespace

namespace b200 {

void set_default_algorithm(Algorithm a) { t_algorithm = a; }
Algorithm default_algorithm() { return env_algorithm(); }

SolveOutcome bicgstab_solve(const CsrMatrix& a, const DenseVector& b, const DenseVector& x0, double tol,
                            std::size_t max_iter, const ReductionPlan& reduction) {
    return single_system(Algorithm::JacobiBiCGStab, a, b, x0, tol, max_iter, reduction);
}

// simulate.cpp:72-178 with every per-cell array in HBM (bc_simulate).
SimulationResult run_simulation(const MechanismSpec& mech, const SimulationConfig& config,
                                const std::vector<CellState>& initial_states) {
    if (config.cells == 0) throw std::invalid_argument("run_simulation: cells must be >= 1");
    if (!(config.dt_seconds > 0.0)) throw std::invalid_argument("run_simulation: dt must be positive");
    if (initial_states.size() != config.cells)
        throw std::invalid_argument("run_simulation: one initial state per cell");
    for (const CellState& st : initial_states)
        if (st.concentrations.size() != mech.n_species)
            throw std::invalid_argument("run_simulation: state dimension mismatch");
    mech.check_invariants();  // as MechanismEvaluator's construction does

    // the mechanism as flat arrays -> the evaluator tables (blockcells_workload.h)
    const std::size_t R = mech.reactions.size(), S = mech.n_species, C = config.cells;
    std::vector<int32_t> kind(R), rptr(R + 1, 0), rlist, pptr(R + 1, 0), plist;
    std::vector<double> coeff(R), texp(R);
    for (std::size_t j = 0; j < R; ++j) {
        const Reaction& r = mech.reactions[j];
        kind[j] = r.kind == ReactionKind::Emission ? 0 : r.kind == ReactionKind::Unimolecular ? 1 : 2;
        for (std::size_t x : r.reactants) rlist.push_back(static_cast<int32_t>(x));
        for (std::size_t x : r.products) plist.push_back(static_cast<int32_t>(x));
        rptr[j + 1] = static_cast<int32_t>(rlist.size());
        pptr[j + 1] = static_cast<int32_t>(plist.size());
        coeff[j] = r.rate_coeff;
        texp[j] = r.temp_exponent;
    }
    bcw_mechanism* m = nullptr;
    if (bcw_mechanism_from_reactions(static_cast<int64_t>(S), static_cast<int64_t>(R), kind.data(), rptr.data(),
                                     rlist.data(), pptr.data(), plist.data(), coeff.data(), texp.data(), &m) != 0)
        throw std::invalid_argument("run_simulation: bad mechanism");
    std::unique_ptr<bcw_mechanism, void (*)(bcw_mechanism*)> hold(m, bcw_mechanism_destroy);
    const int64_t nnz = bcw_nnz(m), nstamps = bcw_stamp_count(m);
    std::vector<int32_t> row_ptr(S + 1), col_idx(static_cast<size_t>(nnz));
    bcw_pattern(m, row_ptr.data(), col_idx.data());
    std::vector<int32_t> sptr(R + 1), sslot(std::max<int64_t>(nstamps, 1)), sother(std::max<int64_t>(nstamps, 1)),
        rp2(R + 1), re2(2 * R + 1), pp2(R + 1), pr2(2 * R + 1), diag(S);
    std::vector<double> ssign(std::max<int64_t>(nstamps, 1));
    bcw_stamp_program(m, sptr.data(), sslot.data(), ssign.data(), sother.data(), rp2.data(), re2.data(), pp2.data(),
                      pr2.data(), diag.data());
    std::vector<double> rates(C * R);
    const int mode = config.mode == ConditionMode::Ideal ? BCW_MODE_IDEAL : BCW_MODE_REALISTIC;
    if (R > 0) bcw_rate_constants(m, 0, static_cast<int64_t>(C), static_cast<int64_t>(C), mode, rates.data(), 0);

    bc_mechanism_tables t{};
    t.species = static_cast<int32_t>(S);
    t.reactions = static_cast<int32_t>(R);
    t.nnz = static_cast<int32_t>(nnz);
    t.stamps = static_cast<int32_t>(nstamps);
    t.row_ptr = row_ptr.data();
    t.col_idx = col_idx.data();
    t.stamp_ptr = sptr.data();
    t.stamp_slot = sslot.data();
    t.stamp_other = sother.data();
    t.stamp_sign = ssign.data();
    t.reactant_ptr = rp2.data();
    t.reactants = re2.data();
    t.product_ptr = pp2.data();
    t.products = pr2.data();
    t.diag_slot = diag.data();

    bc_sim_params prm{};
    prm.cells = static_cast<int64_t>(C);
    prm.steps = static_cast<int64_t>(config.steps);
    prm.dt_seconds = config.dt_seconds;
    prm.tol = config.tol;
    prm.max_iter = static_cast<int64_t>(config.max_iter);
    const Strategy kd = config.solver.strategy.kind;
    prm.strategy = kd == Strategy::OneCell     ? BC_STRATEGY_ONE_CELL
                   : kd == Strategy::MultiCells ? BC_STRATEGY_MULTI_CELLS
                                                : BC_STRATEGY_BLOCK_CELLS;
    prm.algo = env_algorithm() == Algorithm::JacobiBiCGStab ? BC_ALGO_BICGSTAB_JACOBI : BC_ALGO_BICG;
    prm.cells_per_block = config.solver.strategy.cells_per_block
                              ? static_cast<int64_t>(*config.solver.strategy.cells_per_block)
                              : 0;
    prm.max_threads_per_block = static_cast<int64_t>(config.device.max_threads_per_block);
    prm.use_direct_reference = config.solver.use_direct_reference ? 1 : 0;
    prm.newton_rtol = config.newton_rtol;
    prm.max_newton_iterations = static_cast<int64_t>(config.max_newton_iterations);

    std::vector<double> y(C * S);
    for (std::size_t c = 0; c < C; ++c)
        std::copy(initial_states[c].concentrations.begin(), initial_states[c].concentrations.end(), y.begin() + c * S);
    std::vector<bc_step_stats> steps(std::max<std::size_t>(config.steps, 1));
    int64_t abort_step = -1;
    bc_ctx* ctx = context();
    const int st = bc_simulate(ctx, &prm, &t, rates.data(), y.data(), steps.data(), &abort_step);
    if (st == BC_ERR_SOLVER_ABORT)
        throw SolverAbort(static_cast<std::size_t>(abort_step),
                          "non-finite concentration at step " + std::to_string(abort_step));
    if (st != BC_OK) raise_status(st, bc_last_error(ctx));

    SimulationResult out;
    out.final_states.resize(C);
    for (std::size_t c = 0; c < C; ++c) out.final_states[c].concentrations.assign(y.begin() + c * S, y.begin() + (c + 1) * S);
    for (std::size_t i = 0; i < config.steps; ++i) {
        StepStats q;
        q.step = static_cast<std::size_t>(steps[i].step);
        q.newton_iterations = static_cast<std::size_t>(steps[i].newton_iterations);
        q.iterations_effective = static_cast<std::size_t>(steps[i].iterations_effective);
        q.iterations_sum = static_cast<std::size_t>(steps[i].iterations_sum);
        q.max_residual_rms = steps[i].max_residual_rms;
        q.wall_time_ns = steps[i].wall_time_ns;
        q.breakdown_fallbacks = static_cast<std::size_t>(steps[i].breakdown_fallbacks);
        q.clip_events = static_cast<std::size_t>(steps[i].clip_events);
        out.per_step.push_back(q);
    }
    return out;
}

}  // namespace b200

// ---- strategies.cpp surface ------------------------------------------------

void BatchedSystem::check() const {  // strategies.cpp:91-107
    if (cells == 0) throw std::invalid_argument("batched system: no cells");
    if (species == 0) throw std::invalid_argument("batched system: no species");
    if (per_cell_matrices.size() != cells || per_cell_rhs.size() != cells)
        throw std::invalid_argument("batched system: per-cell arrays mismatch");
    const CsrMatrix& first = per_cell_matrices.front();
    for (const CsrMatrix& m : per_cell_matrices) {
        if (m.n_rows != species || m.n_cols != species)
            throw std::invalid_argument("batched system: cell matrix dimension");
        if (m.row_ptr != first.row_ptr || m.col_idx != first.col_idx)
            throw std::invalid_argument("batched system: cells do not share one sparsity pattern");
    }
    for (const DenseVector& b : per_cell_rhs)
        if (b.size() != species) throw std::invalid_argument("batched system: rhs dimension");
}

std::string StrategyConfig::label() const {
    switch (kind) {
        case Strategy::OneCell: return "one-cell";
        case Strategy::MultiCells: return "multi-cells";
        case Strategy::BlockCells:
            return cells_per_block ? "block-cells(" + std::to_string(*cells_per_block) + ")" : "block-cells(N)";
    }
    return "?";
}

AssembledSystem assemble_block_diagonal(const BatchedSystem& system, IndexRange cell_range) {
    if (cell_range.size() == 0) throw std::invalid_argument("assemble_block_diagonal: empty cell range");
    if (cell_range.end > system.cells) throw std::invalid_argument("assemble_block_diagonal: range out of bounds");
    const std::size_t s = system.species;
    AssembledSystem out;
    out.a.n_rows = out.a.n_cols = cell_range.size() * s;
    out.a.row_ptr.push_back(0);
    for (std::size_t c = cell_range.begin; c < cell_range.end; ++c) {
        const CsrMatrix& m = system.per_cell_matrices[c];
        const std::size_t shift = (c - cell_range.begin) * s;
        for (std::size_t i = 0; i < s; ++i) {
            for (std::size_t j = m.row_ptr[i]; j < m.row_ptr[i + 1]; ++j) {
                out.a.col_idx.push_back(m.col_idx[j] + shift);
                out.a.values.push_back(m.values[j]);
            }
            out.a.row_ptr.push_back(out.a.col_idx.size());
        }
        out.b.insert(out.b.end(), system.per_cell_rhs[c].begin(), system.per_cell_rhs[c].end());
    }
    return out;
}

SolveReport solve_one_cell(const BatchedSystem& system, double tol, std::size_t max_iter,
                           const DeviceSpec& device) {
    return run_gpu(system, BC_STRATEGY_ONE_CELL, std::nullopt, device, tol, max_iter, Strategy::OneCell);
}

namespace {
// run_strategy's worker_count reaches the packing threads of One-cell too
SolveReport solve_one_cell_workers(const BatchedSystem& system, double tol, std::size_t max_iter,
                                   const DeviceSpec& device, std::size_t workers) {
    return run_gpu(system, BC_STRATEGY_ONE_CELL, std::nullopt, device, tol, max_iter, Strategy::OneCell, workers);
}
}  // namespace

SolveReport solve_multi_cells(const BatchedSystem& system, const DeviceSpec& device, double tol,
                              std::size_t max_iter) {
    return run_gpu(system, BC_STRATEGY_MULTI_CELLS, std::nullopt, device, tol, max_iter, Strategy::MultiCells);
}

SolveReport solve_block_cells(const BatchedSystem& system, std::optional<std::size_t> cells_per_block,
                              const DeviceSpec& device, double tol, std::size_t max_iter,
                              std::size_t worker_count) {
    return run_gpu(system, BC_STRATEGY_BLOCK_CELLS, cells_per_block, device, tol, max_iter, Strategy::BlockCells,
                   worker_count);
}

SolveReport run_strategy(const BatchedSystem& system, const StrategyConfig& config, const DeviceSpec& device,
                         double tol, std::size_t max_iter, std::size_t worker_count) {
    switch (config.kind) {
        case Strategy::OneCell: return solve_one_cell_workers(system, tol, max_iter, device, worker_count);
        case Strategy::MultiCells: return solve_multi_cells(system, device, tol, max_iter);
        case Strategy::BlockCells:
            return solve_block_cells(system, config.cells_per_block, device, tol, max_iter, worker_count);
    }
    throw std::invalid_argument("run_strategy: unknown strategy");
}

double iteration_reduction_ratio(const SolveReport& a, const SolveReport& b) {
    if (a.iterations_effective == 0) throw std::invalid_argument("iteration_reduction_ratio: zero denominator");
    return static_cast<double>(b.iterations_effective) / static_cast<double>(a.iterations_effective);
}

// ---- bicg.cpp surface -------------------------------------------------------

void BicgWorkspace::resize(std::size_t n, std::size_t n_blocks) {
    r.resize(n);
    r_shadow.resize(n);
    p.resize(n);
    p_shadow.resize(n);
    ap.resize(n);
    atp_shadow.resize(n);
    per_block_error.resize(n_blocks);
}

std::vector<bool> block_converged_mask(const std::vector<double>& per_block_error,
                                       const std::vector<std::size_t>& n_per_block, double tol) {
    if (per_block_error.size() != n_per_block.size())
        throw std::invalid_argument("block_converged_mask: arrays not aligned");
    std::vector<bool> mask(per_block_error.size());
    for (std::size_t b = 0; b < mask.size(); ++b)
        mask[b] = std::sqrt(per_block_error[b] / static_cast<double>(n_per_block[b])) <= tol;
    return mask;
}

SolveOutcome bicg_solve(const CsrMatrix& a, const DenseVector& b, const DenseVector& x0, double tol,
                        std::size_t max_iter, const ReductionPlan& reduction) {
    return single_system(b200::Algorithm::BiCG, a, b, x0, tol, max_iter, reduction);
}

// Every exit of the reference's bicg_solve ends with residual_rms(out.x)
// (bicg.cpp:61-72, 126-141), so its ws.per_block_error holds the per-block
// partials of the fresh residual (b - A x)^2 of the returned x.  x is bit-
// identical here, so the same two reference functions over it (spmv,
// csr.cpp:90-101; plan_reduce_map, reduction.hpp:60-79) give the same bits.
SolveOutcome bicg_solve(const CsrMatrix& a, const DenseVector& b, const DenseVector& x0, double tol,
                        std::size_t max_iter, const ReductionPlan& reduction, BicgWorkspace& ws) {
    SolveOutcome out = single_system(b200::Algorithm::BiCG, a, b, x0, tol, max_iter, reduction);
    const std::size_t n = a.n_rows;
    ws.resize(n, reduction.n_blocks());
    spmv(a, out.x, ws.ap);
    plan_reduce_map(
        n,
        [&](std::size_t i) {
            const double ri = b[i] - ws.ap[i];
            return ri * ri;
        },
        reduction, ws.tree_scratch, std::span<double>(ws.per_block_error));
    return out;
}

}  // namespace blockcells
