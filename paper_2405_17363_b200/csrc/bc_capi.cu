// bc_capi.cu -- C ABI (include/blockcells_b200.h): validation mirroring the
// reference's exceptions, group planning (plan_kernel / solve_block_cells),
// device memory, kernel launches, the LU fallback and merge_groups.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bc_block.cuh"
#include "bc_lu.cuh"
#include "bc_lu_sm.cuh"
#include "bc_multi.cuh"
#include "bc_newton.cuh"
#include "bc_thread.cuh"
#include "bc_tmem.cuh"
#include "bc_latency.cuh"
#include "bc_plan.hpp"
#include "blockcells_b200.h"

namespace {

constexpr int kMaxDynSmem = 227 * 1024;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        const cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Status(BC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device address of page-locked host memory (cudaHostAlloc / cudaHostRegister),
// or nullptr for pageable or device memory.
void* mapped_host_ptr(const void* p) {
    cudaPointerAttributes a;
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

using BlockFn = void (*)(bc::BlockParams);

struct KernelCfg {
    int W, R, RV;
    BlockFn fn[2];
};

#define BC_CFG(W, R, RV) \
    {W, R, RV, {&bc::block_cells_kernel<bc::kBiCG, W, R, RV>, &bc::block_cells_kernel<bc::kBiCGStab, W, R, RV>}}

const KernelCfg kConfigs[] = {
    BC_CFG(1, 1, 1), BC_CFG(1, 2, 2), BC_CFG(1, 4, 4), BC_CFG(1, 8, 5), BC_CFG(1, 8, 8),
    BC_CFG(2, 8, 5), BC_CFG(2, 8, 8), BC_CFG(4, 8, 5), BC_CFG(4, 8, 8), BC_CFG(8, 8, 5),
    BC_CFG(8, 8, 8),
};

const KernelCfg* pick_config(const bc::Geometry& g) {
    const KernelCfg* best = nullptr;
    for (const KernelCfg& k : kConfigs)
        if (k.W == g.W && k.R == g.R && k.RV >= g.RV && (!best || k.RV < best->RV)) best = &k;
    return best;
}

}  // namespace

// Latency-mode row tables of a group geometry (bc_latency.cuh): [lmax][P]
// value indices and gather byte offsets of each thread's row (and, for BiCG,
// of its A^T row); device copies live in the context's plan buffers.
struct LatPlan {
    int P = 0, T = 0, L = 0, xslots = 0, model = 0;
    bool ok = false;
    int32_t *rowof = nullptr, *steps = nullptr, *rvi = nullptr, *tvi = nullptr, *didx = nullptr;
    uint16_t *rxo = nullptr, *txo = nullptr;
};

struct bc_ctx {
    int device = 0;
    int sms = 0;
    std::string err;
    bool has_pattern = false;
    bc::Pattern pat;
    DevBuf d_rp, d_ci;
    DevBuf m_trp, m_trow, m_tval, m_diag, m_ranges, m_work, m_part, m_out;  // Multi-cells
    bool m_ready = false;
    std::map<std::pair<int, int>, bc::GroupPlan> plans;  // (k, with_transpose)
    std::vector<DevBuf> plan_bufs;
    DevBuf values, rhs, x, giters, grms, gflags, counters, lu_scratch, lu_entries, lu_status,
        f_scratch, lu_rms_scratch, lu_chain, t_values, t_work;
    // device-resident simulation (bc_simulate)
    DevBuf sim_tabs, sim_sign, sim_rates, sim_y, sim_prev, sim_values, sim_rhs, sim_dx, sim_red;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    // host-input pipeline: chunk copies + ready flags on copy_st, gated kernels on st
    cudaStream_t copy_st = nullptr;
    cudaEvent_t pipe_ev[2] = {nullptr, nullptr};
    DevBuf pipe_flags;                  // kPipeFlags ready flags + 1 error word
    unsigned int* h_ones = nullptr;     // pinned source of the flag writes
    int64_t launches = 0;
    int32_t kernels = 0;  // BC_KERNEL_* bits since the last bc_solve started
    double model_spmv_wf = 0.0;  // modelled shared wavefronts per group-iteration of the last TMEM launch
    std::map<std::pair<int, int>, struct LatPlan> lat_plans;  // (k, bicg): latency-mode row tables
    std::map<BlockFn, bool> smem_set;
};

namespace {

thread_local std::string g_last_error;  // errors of context-free calls

void set_err(bc_ctx* ctx, const std::string& m) {
    g_last_error = m;
    if (ctx) ctx->err = m;
}

template <class F>
int guarded(bc_ctx* ctx, F&& f) {
    try {
        if (ctx) {
            ctx->err.clear();
            check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
        }
        return f();
    } catch (const Status& s) {
        set_err(ctx, s.what());
        return s.code;
    } catch (const std::bad_alloc&) {
        set_err(ctx, "out of host memory");
        return BC_ERR_NO_MEMORY;
    } catch (const std::exception& e) {
        set_err(ctx, e.what());
        return BC_ERR_INVALID_ARGUMENT;
    }
}

void fail(int code, const std::string& m) { throw Status(code, m); }

bc::Pattern make_pattern(int32_t species, const int32_t* row_ptr, const int32_t* col_idx) {
    if (species < 1) fail(BC_ERR_INVALID_ARGUMENT, "batched system: no species");
    if (!row_ptr || !col_idx) fail(BC_ERR_INVALID_ARGUMENT, "pattern: null pointer");
    bc::Pattern p;
    p.species = species;
    p.row_ptr.assign(row_ptr, row_ptr + species + 1);
    if (p.row_ptr[0] != 0) fail(BC_ERR_INVALID_ARGUMENT, "csr: row_ptr[0] != 0");
    for (int i = 0; i < species; ++i)
        if (p.row_ptr[i] > p.row_ptr[i + 1]) fail(BC_ERR_INVALID_ARGUMENT, "csr: row_ptr decreasing");
    p.nnz = p.row_ptr[species];
    p.col_idx.assign(col_idx, col_idx + p.nnz);
    p.diag.assign(species, -1);
    for (int i = 0; i < species; ++i)
        for (int e = p.row_ptr[i]; e < p.row_ptr[i + 1]; ++e) {
            if (p.col_idx[e] < 0 || p.col_idx[e] >= species)
                fail(BC_ERR_INVALID_ARGUMENT, "csr: column index out of range");
            if (e > p.row_ptr[i] && p.col_idx[e - 1] >= p.col_idx[e])
                fail(BC_ERR_INVALID_ARGUMENT, "csr: columns not strictly increasing within a row");
            if (p.col_idx[e] == i) p.diag[i] = e;
        }
    return p;
}

template <class T>
T* upload(bc_ctx* ctx, const std::vector<T>& v) {
    ctx->plan_bufs.emplace_back();
    DevBuf& b = ctx->plan_bufs.back();
    check_cuda(b.ensure(sizeof(T) * std::max<size_t>(v.size(), 1)), "cudaMalloc(plan)");
    if (!v.empty())
        check_cuda(cudaMemcpy(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice),
                   "cudaMemcpy(plan)");
    return b.as<T>();
}

bc::GroupPlan& get_plan(bc_ctx* ctx, const bc::Pattern& pat, int k, bool with_t,
                        std::map<std::pair<int, int>, bc::GroupPlan>* cache) {
    const auto key = std::make_pair(k, with_t ? 1 : 0);
    auto it = cache->find(key);
    if (it != cache->end()) return it->second;
    bc::GroupPlan gp = bc::build_group_plan(pat, k, with_t);
    gp.d_words = upload(ctx, gp.a.words);
    gp.d_vpos = upload(ctx, gp.a.vpos);
    gp.d_dpos = upload(ctx, gp.dpos);
    gp.d_vidx = upload(ctx, gp.a.vidx);
    gp.d_didx = upload(ctx, gp.didx);
    gp.d_xpos = upload(ctx, gp.a.xpos);
    if (with_t) {
        gp.d_txpos = upload(ctx, gp.at.xpos);
        gp.d_twords = upload(ctx, gp.at.words);
        gp.d_tvpos = upload(ctx, gp.at.vpos);
        gp.d_tvidx = upload(ctx, gp.at.vidx);
    }
    return cache->emplace(key, std::move(gp)).first->second;
}

struct LaunchShape {
    int teams = 1, blocks = 1, threads = 32;
    size_t smem = 0;
    int team_doubles = 0, sched_words = 0, level = 0;
};

LaunchShape choose_shape(bc_ctx* ctx, BlockFn fn, const bc::GroupPlan& gp, bool bicg, int groups) {
    const int W = gp.geo.W, LW = 32 * W;
    const int n_pad = (gp.geo.n + 31) & ~31;
    cudaFuncAttributes fa;
    check_cuda(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes");
    const size_t dyn_max = static_cast<size_t>(kMaxDynSmem) - fa.sharedSizeBytes;
    if (!ctx->smem_set[fn]) {
        check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn_max)),
                   "cudaFuncSetAttribute");
        ctx->smem_set[fn] = true;
    }
    const int sched = gp.a.steps * LW + (bicg ? gp.at.steps * LW : 0);
    const int xa = (gp.a.xslots + 31) & ~31, xt = bicg ? (gp.at.xslots + 31) & ~31 : 0;
    const int vecs = xa + n_pad + (bicg ? xt + n_pad : 0) + (W > 1 ? 8 * W * 32 : 0);
    for (int level = 0; level <= 2; ++level) {
        LaunchShape sh;
        sh.level = level;
        sh.sched_words = level == 0 ? ((sched + 3) & ~3) : 0;
        sh.team_doubles = (level < 2 ? sched : 0) + vecs;
        // Maximise concurrently resident groups (capped by the work available);
        // ties go to fewer teams per CTA, which spreads small batches over more SMs.
        int64_t best = -1;
        const int gmax = std::min(W > 1 ? 15 : 32, 256 / LW);
        for (int G = 1; G <= gmax; ++G) {
            const size_t smem = sizeof(uint32_t) * sh.sched_words + sizeof(double) * G * sh.team_doubles;
            if (smem > dyn_max) break;
            int nb = 0;
            check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, G * LW, smem),
                       "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
            const int64_t conc = std::min<int64_t>(groups, static_cast<int64_t>(nb) * G * ctx->sms);
            if (nb > 0 && conc > best) {
                best = conc;
                sh.teams = G;
                sh.smem = smem;
                sh.blocks = nb;
            }
        }
        if (best <= 0) continue;
        sh.threads = sh.teams * LW;
        const int need = (groups + sh.teams - 1) / sh.teams;
        sh.blocks = std::max(1, std::min(need, sh.blocks * ctx->sms));
        return sh;
    }
    fail(BC_ERR_INVALID_ARGUMENT, "group does not fit in shared memory");
    return LaunchShape{};
}

using TmemFn = void (*)(bc::TmemParams);

// Host-input pipeline (bc_solve): chunks per span, and the smallest batch worth it.
constexpr int kPipeChunksMax = 64;          // per span
constexpr int kPipeFlags = 2 * kPipeChunksMax;  // Block-cells has at most two spans
int pipe_chunks() {  // BC_PIPE_CHUNKS overrides the default 32
    const char* e = std::getenv("BC_PIPE_CHUNKS");
    const int c = e ? std::atoi(e) : 32;
    return std::max(1, std::min(kPipeChunksMax, c));
}
constexpr int64_t kPipeMinCells = 4096;

struct TmemCfg {
    int T, R, RV, warps, ST, CP, ALGO;  // team width (warps per group), tree slots, row slots, warps per CTA,
    TmemFn fn;                          // row streams, gather copies, bc::AlgoKind
};

// Jacobi-BiCGSTAB: one warp per cell at 16 warps/SM (<= 128 registers) or 8
// (<= 255); two-warp teams for schedules too long for 4 cells per lane
// quarter (the scaled mechanism, 312 species: 16 warps = 8 cells/SM instead
// of 8 warps = 8 cells); four-warp teams for latency (BC_TMEM_TEAM=4).
// BiCG runs its pair schedule (A and A^T in one pass, twice as long).
#define BC_TMEM_CFG(T, R, RV, W, ST, CP, A) \
    { T, R, RV, W, ST, CP, A, &bc::block_cells_tmem_kernel<T, R, RV, 32 * W, ST, CP, A> }
constexpr int kS = bc::kBiCGStab, kB = bc::kBiCG;
const TmemCfg kTmemConfigs[] = {
    // BiCGSTAB, one warp per cell
    BC_TMEM_CFG(1, 8, 5, 16, 2, 2, kS), BC_TMEM_CFG(1, 8, 5, 16, 2, 1, kS), BC_TMEM_CFG(1, 8, 5, 16, 1, 2, kS),
    BC_TMEM_CFG(1, 8, 5, 16, 1, 1, kS), BC_TMEM_CFG(1, 8, 8, 16, 2, 2, kS), BC_TMEM_CFG(1, 4, 4, 16, 2, 2, kS),
    BC_TMEM_CFG(1, 16, 10, 8, 2, 2, kS), BC_TMEM_CFG(1, 16, 10, 8, 2, 1, kS),
    // BiCGSTAB, teams
    BC_TMEM_CFG(2, 8, 5, 16, 2, 2, kS), BC_TMEM_CFG(2, 4, 3, 16, 2, 2, kS), BC_TMEM_CFG(4, 2, 2, 16, 1, 2, kS),
    BC_TMEM_CFG(4, 4, 3, 16, 1, 2, kS),
    // BiCG (pair schedules)
    BC_TMEM_CFG(1, 8, 5, 8, 2, 2, kB), BC_TMEM_CFG(1, 8, 5, 8, 2, 1, kB), BC_TMEM_CFG(1, 8, 8, 8, 2, 2, kB),
    BC_TMEM_CFG(1, 4, 4, 8, 2, 2, kB), BC_TMEM_CFG(1, 16, 10, 4, 2, 2, kB), BC_TMEM_CFG(2, 8, 5, 8, 2, 2, kB),
    BC_TMEM_CFG(2, 4, 3, 16, 2, 2, kB),
    // four-warp teams for coupled Block-cells(k) groups of up to 1024 rows
    // (Block-cells(N) at M156: 936 rows, 2 groups per SM)
    BC_TMEM_CFG(4, 8, 5, 8, 1, 2, kS), BC_TMEM_CFG(4, 8, 8, 8, 1, 2, kS), BC_TMEM_CFG(4, 8, 8, 8, 2, 2, kS),
    BC_TMEM_CFG(4, 8, 5, 4, 2, 2, kB),
    BC_TMEM_CFG(4, 8, 8, 4, 2, 2, kB),
};
#undef BC_TMEM_CFG

int tmem_warps_pref() {
    const char* e = std::getenv("BC_TMEM_WARPS");
    return e ? std::atoi(e) : 16;
}

bool tmem_disabled() {
    const char* e = std::getenv("BC_KERNEL");
    return e && std::string(e) == "v1";
}

// The TMEM kernel (bc_tmem.cuh): BiCG or Jacobi-BiCGSTAB, one warp per group, schedule
// words + per-group values resident in Tensor Memory.  Returns false when the
// group does not qualify (the caller then uses the v1 kernel).
// Largest sigma with sqrt(sigma / n) <= tol, both correctly rounded (x86-64
// SSE2 here, __dsqrt_rn/__ddiv_rn on the GPU), so that the kernel's test
// sigma <= sigma_max decides exactly as bicg.cpp:84/129 does.  The predicate
// is monotone in sigma, so a bisection over the ordered bit patterns of
// non-negative doubles finds the boundary.
double sigma_threshold(double tol, int n) {
    auto ok = [&](double s) { return std::sqrt(s / static_cast<double>(n)) <= tol; };
    uint64_t lo = 0, hi = 0x7FF0000000000000ull;  // ok(+0) is true (tol > 0)
    double dhi;
    std::memcpy(&dhi, &hi, 8);
    if (ok(dhi)) return dhi;  // tol = +inf
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        double dm;
        std::memcpy(&dm, &mid, 8);
        (ok(dm) ? lo : hi) = mid;
    }
    double r;
    std::memcpy(&r, &lo, 8);
    return r;
}

// The TMEM kernel runs a group on a team of 1, 2 or 4 warps whatever the v1
// team width: its reduction tree is Q/team slots per lane (Q <= 16 here).
bool tmem_fits(const bc::GroupPlan& gp) { return gp.geo.P >= 32 && gp.geo.Q <= 32; }

int tmem_team_pref() {
    const char* e = std::getenv("BC_TMEM_TEAM");
    const int t = e ? std::atoi(e) : 0;
    return t == 1 || t == 2 || t == 4 ? t : 0;
}

// Warps per TMEM lane quarter that fit 512 columns: S/2 word columns shared
// by the quarter, 2S value columns per warp (one group, or one team member).
// extra: further columns per warp (BiCGSTAB keeps D^-1 there: 2 per row slot).
int tmem_groups_per_quarter(int S, int extra = 0) {
    return S > 0 ? std::min(4, (512 - S / 2) / (2 * S + extra)) : 0;
}

// The TMEM schedule of a plan for a team width, built and uploaded once.
// BiCG plans (built with the transpose) get the pair schedule: A p and A^T p~
// in one pass.
// quick: fewer annealing moves, for batches too small to be bound by the
// shared-memory pipe.
bc::TmemPlan& tmem_schedule(bc_ctx* ctx, const bc::Pattern& pat, bc::GroupPlan& gp, int team, bool quick) {
    const int key = team + (quick ? 8 : 0);
    auto it = gp.tmem.find(key);
    if (it != gp.tmem.end()) return it->second;
    bc::TmemPlan tp;
    try {
        tp.tm = bc::build_tmem_schedule(pat, gp.k, gp.at.steps > 0, team, true, quick);
    } catch (const std::invalid_argument&) {  // e.g. a gather vector beyond 15-bit offsets
        tp.tm.steps = 0;                       // no schedule: pick_tmem_cfg finds no instance
    }
    tp.d_words = upload(ctx, tp.tm.words);
    tp.d_vidx = upload(ctx, tp.tm.vidx);
    return gp.tmem.emplace(key, std::move(tp)).first->second;
}

// Kernel instance for a schedule: same team and tree width, enough row
// slots, and the most warps the schedule's TMEM footprint allows (capped by
// BC_TMEM_WARPS).
const TmemCfg* pick_tmem_cfg(const bc::GroupPlan& gp, const bc::TmemPlan& tp) {
    const int algo = tp.tm.pair ? bc::kBiCG : bc::kBiCGStab;
    const int T = tp.tm.team;
    const int rv_min = ((gp.geo.n + 31) / 32 + T - 1) / T;
    const int cpq = tmem_groups_per_quarter(tp.tm.steps, algo == bc::kBiCGStab ? 2 * rv_min : 0);
    if (cpq < 1) return nullptr;
    const int want = std::min(4 * cpq, tmem_warps_pref());
    const TmemCfg* cfg = nullptr;
    // among matching instances: the fewest warps >= want (most registers), else the most warps
    auto better = [&](const TmemCfg& t, const TmemCfg* c) {
        if (!c) return true;
        const bool tf = t.warps >= want, cf = c->warps >= want;
        if (tf != cf) return tf;
        if (t.warps != c->warps) return tf ? t.warps < c->warps : t.warps > c->warps;
        return t.RV < c->RV;
    };
    for (const TmemCfg& t : kTmemConfigs) {
        if (t.T != T || t.R * T != gp.geo.Q || t.RV * T < (gp.geo.n + 31) / 32 || t.ST != tp.tm.streams ||
            t.CP != tp.tm.copies || t.ALGO != algo)
            continue;
        if (better(t, cfg)) cfg = &t;
    }
    return cfg;
}

// Team width for a launch of `groups` groups (BC_TMEM_TEAM overrides):
//   * batches that leave SMs idle trade cells in flight for latency: up to
//     4 groups per SM run as four-warp teams, up to 8 as two-warp teams
//     (B200, M156, P regime: 100 cells 30.5k cell-solves/s with four-warp
//     teams vs 20.0k, 1000 cells 163k with two-warp teams vs 148k);
//   * otherwise one warp per cell while 2 cells fit a lane quarter (8
//     warps/SM), else two-warp teams: M312 BiCG's pair schedule (S = 200, 4
//     warps/SM alone) 209k with teams vs 157k at 100k cells; where 2 cells fit,
//     teams lose to their barriers (M312 BiCGSTAB 212k vs 221k, M156 BiCG
//     455k vs 476k, M156 BiCGSTAB 289k vs 502k).
// The first candidate with a kernel instance wins.
bc::TmemPlan* tmem_plan(bc_ctx* ctx, const bc::Pattern& pat, bc::GroupPlan& gp, int groups, const TmemCfg** cfg) {
    if (tmem_disabled() || !tmem_fits(gp)) return nullptr;
    int cand[5], nc = 0;
    if (const int pref = tmem_team_pref()) cand[nc++] = pref;
    if (groups <= 4 * ctx->sms) cand[nc++] = 4;
    else if (groups <= 8 * ctx->sms) cand[nc++] = 2;
    cand[nc++] = 0;  // the default, decided from the one-warp schedule below
    cand[nc++] = 4;  // four-warp teams (coupled groups)
    cand[nc++] = 1;  // last resort: one warp, whatever its lane-quarter occupancy
    const bool quick = groups <= 8 * ctx->sms;
    for (int i = 0; i < nc; ++i) {
        int team = cand[i];
        if (team == 0) {
            if (gp.geo.Q > 16) continue;  // one- and two-warp trees stop at 16 slots per lane
            bc::TmemPlan& one = tmem_schedule(ctx, pat, gp, 1, quick);
            team = tmem_groups_per_quarter(one.tm.steps) >= 2 ? 1 : 2;
        }
        if (gp.geo.Q % team || (team == 1 && gp.geo.Q > 16)) continue;
        bc::TmemPlan& tp = tmem_schedule(ctx, pat, gp, team, quick);
        if (const TmemCfg* c = pick_tmem_cfg(gp, tp)) {
            *cfg = c;
            return &tp;
        }
    }
    return nullptr;
}

// Per-lane owner tables for a kernel instance with RV row slots: copy-0
// gather slot | Y slot << 16, and copy 1's slots two row slots per word; for a
// pair schedule the same again for p~ and the A^T outputs.  Rows >= n go to
// the trash slot (after every copy) and read the zero Y slot.
void ensure_tmem_lane_tables(bc_ctx* ctx, const bc::GroupPlan& gp, bc::TmemPlan& tp, int RV) {
    if (tp.lane_rv == RV) return;
    const bc::TmemSchedule& tm = tp.tm;
    const int n = gp.geo.n, trash = tm.xslots, nx = tm.pair ? 2 * n : n, T = tm.team;
    for (int part = 0; part < (tm.pair ? 2 : 1); ++part) {
        // owner row of (slot j, warp w, lane l) is (j*T + w)*32 + l (team_reduce's layout)
        std::vector<uint32_t> xy(static_cast<size_t>(RV) * T * 32);
        std::vector<uint32_t> x1(static_cast<size_t>((RV + 1) / 2) * T * 32, 0u);
        for (int j = 0; j < RV; ++j)
            for (int w = 0; w < T; ++w)
                for (int l = 0; l < 32; ++l) {
                    const int row = (j * T + w) * 32 + l, col = part * n + row;
                    const bool ok = row < n;
                    xy[row] = static_cast<uint32_t>(ok ? tm.xpos[col] : trash) |
                              (static_cast<uint32_t>(ok ? tm.yslot[col] : tm.yslots) << 16);
                    const uint32_t s1 =
                        static_cast<uint32_t>(ok && tm.copies > 1 ? tm.xpos[static_cast<size_t>(nx) + col] : trash);
                    x1[((j / 2) * T + w) * 32 + l] |= s1 << (16 * (j % 2));
                }
        (part ? tp.d_xyT : tp.d_xy) = upload(ctx, xy);
        (part ? tp.d_x1T : tp.d_x1) = upload(ctx, x1);
    }
    tp.lane_rv = RV;
}

bool launch_tmem(bc_ctx* ctx, const bc::Pattern& pat, bc::GroupPlan& gp, int64_t cell0, int64_t gout0,
                 int groups, const double* values, const double* rhs, double* x, double tol, int64_t max_iter,
                 unsigned int* counter, cudaStream_t st, const bc::InputGate& gate = bc::InputGate{}) {
    const TmemCfg* cfg = nullptr;
    bc::TmemPlan* tpp = tmem_plan(ctx, pat, gp, groups, &cfg);
    if (!tpp) return false;
    bc::TmemPlan& tp = *tpp;
    ensure_tmem_lane_tables(ctx, gp, tp, cfg->RV);
    const int S = tp.tm.steps;
    const int cpq =
        std::min(cfg->warps / 4, tmem_groups_per_quarter(S, cfg->ALGO == bc::kBiCGStab ? 2 * cfg->RV : 0));
    if (cpq < 1) return false;
    const int warps = 4 * cpq, T = cfg->T, teams = warps / T;
    const int xslots = (tp.tm.xslots + 1 + 31) & ~31, yslots = tp.tm.yslots + 32 * T;
    const int xalign = static_cast<int>(bc::padded_len(8 * xslots));
    const size_t smem = sizeof(int32_t) * S * 32 * T + static_cast<size_t>(xalign) * (teams + 1) +
                        sizeof(double) * teams * yslots + (T > 1 ? sizeof(double) * teams * 2 * 4 * 32 * T : 0);
    if (smem > static_cast<size_t>(kMaxDynSmem - 1024)) return false;
    if (!ctx->smem_set[reinterpret_cast<BlockFn>(cfg->fn)]) {
        check_cuda(cudaFuncSetAttribute(cfg->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem - 1024),
                   "cudaFuncSetAttribute(tmem)");
        ctx->smem_set[reinterpret_cast<BlockFn>(cfg->fn)] = true;
    }
    bc::TmemParams p{};
    p.values = values;
    p.rhs = rhs;
    p.x_out = x;
    p.g_iters = ctx->giters.as<int32_t>();
    p.g_rms = ctx->grms.as<double>();
    p.g_flags = ctx->gflags.as<uint8_t>();
    p.words = tp.d_words;
    p.vidx = tp.d_vidx;
    p.didx = gp.d_didx;
    p.lane_xy = tp.d_xy;
    p.lane_x1 = tp.d_x1;
    p.lane_xyT = tp.d_xyT;
    p.lane_x1T = tp.d_x1T;
    p.counter = counter;
    p.cell_offset = cell0;
    p.group_offset = gout0;
    p.group_count = groups;
    p.n = gp.geo.n;
    p.nnz = pat.nnz;
    p.S = S;
    p.P = gp.geo.P;
    p.species = pat.species;
    p.kc = gp.k;
    p.xslots = xslots;
    p.yslots = yslots;
    p.xalign = xalign;
    p.ystream = tp.tm.ystream;
    p.cells_per_quarter = cpq;
    p.sigma_max = sigma_threshold(tol, gp.geo.n);
    p.tol = tol;
    // int loop counter: clamped one below INT_MAX so `++it` cannot overflow.  A
    // cell still iterating after 2^31 - 2 iterations (hours of solve) stops
    // there; per-group iteration counts are int32 in the C ABI anyway.
    p.max_iter = static_cast<int>(std::min<int64_t>(max_iter, 0x7FFFFFFE));
    p.gate = gate;
    const int blocks = std::max(1, std::min(ctx->sms, (groups + teams - 1) / teams));
    check_cuda(cudaMemsetAsync(counter, 0, sizeof(unsigned int), st), "cudaMemsetAsync(counter)");
    cfg->fn<<<blocks, warps * 32, smem, st>>>(p);
    check_cuda(cudaGetLastError(), "block_cells_tmem_kernel launch");
    ctx->launches++;
    ctx->kernels |= BC_KERNEL_TMEM;
    // the planner's bank model: one pass per SpMV (BiCG's pair schedule does A p and A^T p~ in one)
    ctx->model_spmv_wf = static_cast<double>(tp.tm.model_total) * (tp.tm.pair ? 1 : 2);
    return true;
}

// ---- latency mode (bc_latency.cuh) ----------------------------------------

using LatFn = void (*)(bc::LatencyParams);
struct LatCfg {
    int R, RV, LMAX, ALGO;  // tree slots per lane (P/32), warps = row slots per lane, padded row length
    LatFn fn;
};
#define BC_LAT_CFG(R, RV, L, A) {R, RV, L, A, &bc::block_cells_latency_kernel<R, RV, L, A>}
#define BC_LAT_CFGS(R, RV, A) BC_LAT_CFG(R, RV, 16, A), BC_LAT_CFG(R, RV, 24, A), BC_LAT_CFG(R, RV, 32, A)
// P = 64 .. 256; the warps (RV) cover ceil(n/32) row slots -- an instance with
// more warps than rows needs runs the extra rows as zeros.  P = 512 (M312:
// ten warps of ~170 registers, spilling) measured slower than the TMEM
// kernel's two-warp teams at 100 cells (6.74 vs 6.29 ms), so it has none.
const LatCfg kLatConfigs[] = {
    BC_LAT_CFGS(2, 2, kS), BC_LAT_CFGS(4, 4, kS), BC_LAT_CFGS(8, 5, kS), BC_LAT_CFGS(8, 8, kS),
    BC_LAT_CFGS(2, 2, kB), BC_LAT_CFGS(4, 4, kB), BC_LAT_CFGS(8, 5, kB), BC_LAT_CFGS(8, 8, kB),
};
#undef BC_LAT_CFGS
#undef BC_LAT_CFG

// The instance for a group geometry: R = P/32, the fewest warps covering the rows.
const LatCfg* latency_cfg(int64_t n, int lmax, bool bicg) {
    const int64_t P = bc::padded_len(n);
    const int R = static_cast<int>(P / 32), need = static_cast<int>((n + 31) / 32);
    const int L = lmax <= 16 ? 16 : lmax <= 24 ? 24 : 32;
    const LatCfg* best = nullptr;
    for (const LatCfg& c : kLatConfigs)
        if (c.R == R && c.RV >= need && c.LMAX == L && c.ALGO == (bicg ? bc::kBiCG : bc::kBiCGStab) &&
            (!best || c.RV < best->RV))
            best = &c;
    return best;
}

// BC_LATENCY: 0 never, 1 whenever a group qualifies; default: launches of at
// most BC_LATENCY_MAX_GROUPS groups (default one per SM), where the
// throughput kernel would leave SMs idle and one cell's iteration latency is
// the whole run.
bool latency_wanted(const bc_ctx* ctx, int groups) {
    if (const char* e = std::getenv("BC_LATENCY")) {
        if (std::string(e) == "0") return false;
        if (std::string(e) == "1") return true;
    }
    if (tmem_team_pref() || tmem_disabled()) return false;  // an explicit kernel choice
    const char* m = std::getenv("BC_LATENCY_MAX_GROUPS");
    const int mx = m ? std::atoi(m) : ctx->sms;
    return groups <= mx;
}

LatPlan& latency_plan(bc_ctx* ctx, const bc::Pattern& pat, int k, bool bicg) {
    const auto key = std::make_pair(k, bicg ? 1 : 0);
    auto it = ctx->lat_plans.find(key);
    if (it != ctx->lat_plans.end()) return it->second;
    LatPlan lp;
    const int64_t n = static_cast<int64_t>(k) * pat.species;
    const int64_t P = bc::padded_len(n);
    if (P >= 64 && P <= 256) {
        // longest row (BiCG: or A^T row) picks the instance's padded length
        std::vector<int> clen(pat.species, 0);
        int lmax = 0;
        for (int i = 0; i < pat.species; ++i) {
            lmax = std::max(lmax, pat.row_ptr[i + 1] - pat.row_ptr[i]);
            for (int e = pat.row_ptr[i]; e < pat.row_ptr[i + 1]; ++e) clen[pat.col_idx[e]]++;
        }
        if (bicg)
            for (int c : clen) lmax = std::max(lmax, c);
        const LatCfg* cfg = lmax <= 32 ? latency_cfg(n, lmax, bicg) : nullptr;
        if (cfg) {
            try {
                const bc::LatencySchedule ls = bc::build_latency_schedule(pat, k, bicg, 32 * cfg->RV);
                lp.ok = ls.lmax <= 32 && ls.L == cfg->LMAX && ls.T == 32 * cfg->RV;
                lp.P = ls.P;
                lp.T = ls.T;
                lp.L = ls.L;
                lp.xslots = ls.xslots;
                lp.model = ls.model_wavefronts;
                if (lp.ok) {
                    lp.rowof = upload(ctx, ls.rowof);
                    lp.steps = upload(ctx, ls.steps);
                    lp.rvi = upload(ctx, ls.rvi);
                    lp.rxo = upload(ctx, ls.rxo);
                    lp.didx = upload(ctx, ls.didx);
                    if (bicg) {
                        lp.tvi = upload(ctx, ls.tvi);
                        lp.txo = upload(ctx, ls.txo);
                    }
                }
            } catch (const std::invalid_argument&) {
                lp.ok = false;  // offsets beyond 16 bits: the throughput kernels take it
            }
        }
    }
    return ctx->lat_plans.emplace(key, lp).first->second;
}

bool launch_latency(bc_ctx* ctx, const bc::Pattern& pat, const bc::GroupPlan& gp, int algo, int64_t cell0,
                    int64_t gout0, int groups, const double* values, const double* rhs, double* x, double tol,
                    int64_t max_iter, cudaStream_t st, const bc::InputGate& gate = bc::InputGate{}) {
    if (!latency_wanted(ctx, groups)) return false;
    const bool bicg = algo == BC_ALGO_BICG;
    LatPlan& lp = latency_plan(ctx, pat, gp.k, bicg);
    if (!lp.ok) return false;
    const LatCfg* cfg = nullptr;
    for (const LatCfg& c : kLatConfigs)
        if (c.R == lp.P / 32 && 32 * c.RV == lp.T && c.LMAX == lp.L && c.ALGO == (bicg ? bc::kBiCG : bc::kBiCGStab))
            cfg = &c;
    if (!cfg) return false;
    bc::LatencyParams p{};
    p.values = values;
    p.rhs = rhs;
    p.x_out = x;
    p.g_iters = ctx->giters.as<int32_t>();
    p.g_rms = ctx->grms.as<double>();
    p.g_flags = ctx->gflags.as<uint8_t>();
    p.rowof = lp.rowof;
    p.steps = lp.steps;
    p.rvi = lp.rvi;
    p.rxo = lp.rxo;
    p.tvi = lp.tvi;
    p.txo = lp.txo;
    p.didx = lp.didx;
    p.cell_offset = cell0;
    p.group_offset = gout0;
    p.group_count = groups;
    p.n = gp.geo.n;
    p.nnz = pat.nnz;
    p.P = lp.P;
    p.species = pat.species;
    p.kc = gp.k;
    p.xs = lp.xslots;
    p.sigma_max = sigma_threshold(tol, gp.geo.n);
    p.tol = tol;
    p.max_iter = static_cast<int>(std::min<int64_t>(max_iter, 0x7FFFFFFE));
    p.gate = gate;
    // Y [2][P] + the gather region
    const int threads = lp.T;
    const size_t smem = sizeof(double) * (2 * static_cast<size_t>(lp.P) + static_cast<size_t>(lp.xslots));
    if (smem > static_cast<size_t>(kMaxDynSmem - 1024)) return false;
    if (!ctx->smem_set[reinterpret_cast<BlockFn>(cfg->fn)]) {
        check_cuda(cudaFuncSetAttribute(cfg->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem - 1024),
                   "cudaFuncSetAttribute(latency)");
        ctx->smem_set[reinterpret_cast<BlockFn>(cfg->fn)] = true;
    }
    int per_sm = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cfg->fn, threads, smem), "occupancy(latency)");
    const int blocks = std::max(1, std::min(groups, ctx->sms * std::max(1, per_sm)));
    cfg->fn<<<blocks, threads, smem, st>>>(p);
    check_cuda(cudaGetLastError(), "block_cells_latency_kernel launch");
    ctx->launches++;
    ctx->kernels |= BC_KERNEL_LATENCY;
    return true;
}

// Launch the fused kernel over `groups` groups of kc cells starting at cell0.
void launch_block(bc_ctx* ctx, const bc::Pattern& pat, const bc::GroupPlan& gp, int algo,
                  int64_t cell0, int64_t gout0, int groups, const double* values,
                  const double* rhs, const double* x0, double* x, double tol, int64_t max_iter,
                  unsigned int* counter, cudaStream_t st, const bc::InputGate& gate = bc::InputGate{}) {
    const KernelCfg* cfg = pick_config(gp.geo);
    if (!cfg) fail(BC_ERR_INVALID_ARGUMENT, "no kernel configuration for this group size");
    const bool bicg = algo == BC_ALGO_BICG;
    BlockFn fn = cfg->fn[bicg ? 0 : 1];
    const LaunchShape sh = choose_shape(ctx, fn, gp, bicg, groups);
    bc::BlockParams p{};
    p.values = values;
    p.rhs = rhs;
    p.x0 = x0;
    p.x_out = x;
    p.g_iters = ctx->giters.as<int32_t>();
    p.g_rms = ctx->grms.as<double>();
    p.g_flags = ctx->gflags.as<uint8_t>();
    p.words = gp.d_words;
    p.twords = gp.d_twords;
    p.vpos = gp.d_vpos;
    p.tvpos = gp.d_tvpos;
    p.dpos = gp.d_dpos;
    p.counter = counter;
    p.cell_offset = cell0;
    p.group_offset = gout0;
    p.group_count = groups;
    p.n = gp.geo.n;
    p.species = pat.species;
    p.nnz = pat.nnz;
    p.kc = gp.k;
    p.S = gp.a.steps;
    p.St = bicg ? gp.at.steps : 0;
    p.P = gp.geo.P;
    p.teams = sh.teams;
    p.team_doubles = sh.team_doubles;
    p.sched_words = sh.sched_words;
    p.tol = tol;
    p.max_iter = max_iter;
    p.level = sh.level;
    p.gate = gate;
    p.vidx = gp.d_vidx;
    p.tvidx = gp.d_tvidx;
    p.didx = gp.d_didx;
    p.xpos = gp.d_xpos;
    p.txpos = gp.d_txpos;
    p.xslots = (gp.a.xslots + 31) & ~31;
    p.txslots = bicg ? (gp.at.xslots + 31) & ~31 : 0;
    check_cuda(cudaMemsetAsync(counter, 0, sizeof(unsigned int), st), "cudaMemsetAsync(counter)");
    fn<<<sh.blocks, sh.threads, sh.smem, st>>>(p);
    check_cuda(cudaGetLastError(), "block_cells_kernel launch");
    ctx->launches++;
    ctx->kernels |= BC_KERNEL_BLOCK;
}

struct GroupSpan {
    int64_t cell0, gout0;
    int k, count;
};

// plan_kernel (exec_model.cpp:102-161) + the group partition of
// solve_block_cells (strategies.cpp:209-213).
void plan_groups(const bc_solve_params* prm, int species, double* cpb, int64_t* n_groups,
                 std::vector<GroupSpan>* spans) {
    const int64_t mtpb = prm->max_threads_per_block > 0 ? prm->max_threads_per_block : 1024;
    if (prm->cells < 1) fail(BC_ERR_INVALID_ARGUMENT, "batched system: no cells");
    if (species > mtpb)
        fail(BC_ERR_UNSUPPORTED_MECHANISM, "mechanism needs more threads per cell than a block provides");
    int64_t k = 1;
    switch (prm->strategy) {
        case BC_STRATEGY_ONE_CELL:
        case BC_STRATEGY_THREAD_PER_CELL:
            *cpb = 1.0;
            k = 1;
            break;
        case BC_STRATEGY_MULTI_CELLS:
            *cpb = static_cast<double>(mtpb) / static_cast<double>(species);
            *n_groups = 1;
            if (spans) spans->push_back({0, 0, 0, 1});
            return;
        case BC_STRATEGY_BLOCK_CELLS:
            if (prm->cells_per_block > 0) {
                k = prm->cells_per_block;
                if (k * species > mtpb)
                    fail(BC_ERR_INVALID_GROUPING, "requested cells per block exceeds the thread budget");
            } else if (prm->cells_per_block == 0) {
                k = mtpb / species;
            } else {
                fail(BC_ERR_INVALID_ARGUMENT, "plan_kernel: cells per block must be >= 1");
            }
            *cpb = static_cast<double>(k);
            break;
        default:
            fail(BC_ERR_INVALID_ARGUMENT, "run_strategy: unknown strategy");
    }
    const int64_t full = prm->cells / k, rem = prm->cells % k;
    *n_groups = full + (rem ? 1 : 0);
    if (spans) {
        if (full) spans->push_back({0, 0, static_cast<int>(k), static_cast<int>(full)});
        if (rem) spans->push_back({full * k, full, static_cast<int>(rem), 1});
    }
}

}  // namespace

// ---- Multi-cells (bc_multi.cuh) -----------------------------------------

// Transpose tables (per local column, entries in ascending row order) and the
// diagonal of one pattern, uploaded into the given buffers.
void upload_multi_tables(const bc::Pattern& pat, DevBuf* trp, DevBuf* trow, DevBuf* tval, DevBuf* diag) {
    const int s = pat.species;
    std::vector<int32_t> cnt(s + 1, 0), tr(pat.nnz), tv(pat.nnz), dg(s);
    for (int e = 0; e < pat.nnz; ++e) cnt[pat.col_idx[e] + 1]++;
    for (int j = 0; j < s; ++j) cnt[j + 1] += cnt[j];
    std::vector<int32_t> next(cnt.begin(), cnt.end() - 1);
    for (int r = 0; r < s; ++r)
        for (int e = pat.row_ptr[r]; e < pat.row_ptr[r + 1]; ++e) {
            const int q = next[pat.col_idx[e]]++;
            tr[q] = r;
            tv[q] = e;
        }
    for (int r = 0; r < s; ++r) dg[r] = pat.diag[r];
    auto up = [](DevBuf* b, const std::vector<int32_t>& v) {
        check_cuda(b->ensure(sizeof(int32_t) * std::max<size_t>(v.size(), 1)), "cudaMalloc(multi)");
        if (!v.empty())
            check_cuda(cudaMemcpy(b->p, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice), "H2D multi");
    };
    up(trp, cnt);
    up(trow, tr);
    up(tval, tv);
    up(diag, dg);
}

// LU fallback (bc_lu.cuh) for the listed groups; throws SingularMatrix.
// g_rms == nullptr: solutions only (the caller computes the residual).
// Coupled groups are factored block by block (mode 0); a group with a non-
// finite input or result is rerun densely (mode 1), like one-cell groups.
void run_lu(bc_ctx* ctx, const std::vector<bc::LuEntry>& ents, const double* d_values, const double* d_rhs,
            double* d_x, double* g_rms, int s, int nnz, int block_width, cudaStream_t st, int mode = 0,
            uint8_t* d_chain_flags = nullptr, int conv = 0, int flip = 0, int later_neg = 0) {
    int64_t nmax = 0, kmax = 0;
    for (const auto& e : ents) {
        nmax = std::max<int64_t>(nmax, static_cast<int64_t>(e.kc) * s);
        kmax = std::max<int64_t>(kmax, e.kc);
    }
    if (nmax > bc::kMaxGroupRows) fail(BC_ERR_INVALID_ARGUMENT, "LU fallback group exceeds 2048 rows");
    const bool blockdiag = mode == 0 && kmax > 1;
    const int64_t stride = blockdiag ? kmax * s * s : nmax * nmax;
    const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(ents.size()),
                                                                 (int64_t(1) << 31) / (stride * 8)));
    check_cuda(ctx->lu_scratch.ensure(sizeof(double) * stride * batch), "cudaMalloc(lu)");
    check_cuda(ctx->lu_entries.ensure(sizeof(bc::LuEntry) * ents.size()), "cudaMalloc");
    check_cuda(ctx->lu_status.ensure(sizeof(int32_t) * ents.size()), "cudaMalloc");
    check_cuda(ctx->lu_rms_scratch.ensure(sizeof(double) * (ents.size() + 1)), "cudaMalloc");
    std::vector<bc::LuEntry> dev_ents = ents;
    if (!g_rms)  // park the per-group residuals in scratch
        for (size_t i = 0; i < dev_ents.size(); ++i) dev_ents[i].gout = static_cast<int64_t>(i);
    check_cuda(cudaMemcpyAsync(ctx->lu_entries.p, dev_ents.data(), sizeof(bc::LuEntry) * dev_ents.size(),
                               cudaMemcpyHostToDevice, st), "H2D lu entries");
    const int64_t pmax = bc::padded_len(nmax);
    // panels in shared memory while a panel of the largest factored matrix fits in 48 KB
    const int64_t prow = blockdiag ? s : nmax;
    const int panel_rows = prow * (bc::kLuPanel + 1) * 8 <= 48 * 1024 ? static_cast<int>(prow) : 0;
    // [panel] perm | sum (n) | ycopy (n) | slots (max(padded n, n, 8 warps x species))
    size_t smem = sizeof(double) * panel_rows * (bc::kLuPanel + 1) + sizeof(int) * ((nmax + 1) & ~1) +
                  sizeof(double) * (2 * nmax + std::max<int64_t>(std::max(pmax, nmax), 8 * s));
    // opt in above 48 KB of static + dynamic shared memory (per device: set on every call)
    cudaFuncAttributes fa{};
    check_cuda(cudaFuncGetAttributes(&fa, bc::lu_fallback_kernel), "cudaFuncGetAttributes(lu)");
    const int lu_dyn_max = kMaxDynSmem - static_cast<int>(fa.sharedSizeBytes);
    check_cuda(cudaFuncSetAttribute(bc::lu_fallback_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lu_dyn_max),
               "cudaFuncSetAttribute(lu)");
    // BC_LU_SMEM=1: block-diagonal groups whose s x s block fits are factored in
    // shared memory (one CTA per SM).  Measured slower than three scratch-resident
    // CTAs per SM (B200, Block-cells(N) M156 P, 100k cells: 557 vs 384 ms):
    // the kernel is bound by its serial chains, which more CTAs overlap.
    const size_t smem_blk = sizeof(int) * ((nmax + 1) & ~1) +
                            sizeof(double) * (2 * nmax + std::max<int64_t>(pmax, static_cast<int64_t>(s) * s));
    const char* lue = std::getenv("BC_LU_SMEM");
    const bool use_smem_block = blockdiag && smem_blk <= static_cast<size_t>(lu_dyn_max) && lue && *lue == '1';
    if (use_smem_block) smem = smem_blk;
    if (smem > static_cast<size_t>(lu_dyn_max)) fail(BC_ERR_INVALID_ARGUMENT, "LU fallback: group too large");
    // Blocks that fit in shared memory (bc_lu_sm.cuh): factor kernel + solve
    // kernel.  Not for the explicit dense reruns and the Multi-cells chain links.
    const char* lsm = std::getenv("BC_LU_SM");
    const bool use_sm = !use_smem_block && mode == 0 && !d_chain_flags && !conv && !flip && !later_neg &&
                        s <= bc::kLuSmMaxRows && kmax <= 32 * 32 &&
                        bc::lu_sm_factor_smem(s) + 1024 <= static_cast<size_t>(kMaxDynSmem) && !(lsm && *lsm == '0');
    const int sm_warps = static_cast<int>(std::min<int64_t>(kmax, 32));
    const size_t sm_solve_smem = bc::lu_sm_solve_smem(nmax, pmax, sm_warps, s);
    if (use_sm) {
        static_assert(sizeof(bc::LuEntry) == 24, "LuEntry layout");
        check_cuda(cudaFuncSetAttribute(bc::lu_sm_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(bc::lu_sm_factor_smem(s))),
                   "cudaFuncSetAttribute(lu_sm_factor)");
        check_cuda(cudaFuncSetAttribute(bc::lu_sm_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kMaxDynSmem - 1024),
                   "cudaFuncSetAttribute(lu_sm_solve)");
        if (sm_solve_smem > static_cast<size_t>(kMaxDynSmem - 1024))
            fail(BC_ERR_INVALID_ARGUMENT, "LU fallback: group too large");
    }
    for (size_t b0 = 0; b0 < ents.size(); b0 += batch) {
        const int cnt = static_cast<int>(std::min<int64_t>(batch, ents.size() - b0));
        bc::LuParams lp{};
        lp.values = d_values;
        lp.rhs = d_rhs;
        lp.x_out = d_x;
        lp.g_rms = g_rms ? g_rms : ctx->lu_rms_scratch.as<double>();
        lp.status = ctx->lu_status.as<int32_t>() + b0;
        lp.entries = ctx->lu_entries.as<bc::LuEntry>() + b0;
        lp.row_ptr = ctx->d_rp.as<int32_t>();
        lp.col_idx = ctx->d_ci.as<int32_t>();
        lp.scratch = ctx->lu_scratch.as<double>();
        lp.stride = stride;
        lp.species = s;
        lp.nnz = nnz;
        lp.block_width = block_width;
        lp.mode = blockdiag ? 0 : 1;
        lp.panel_rows = panel_rows;
        lp.smem_block = use_smem_block ? 1 : 0;
        lp.conv = conv;
        lp.flip = flip;
        lp.later_neg = later_neg;
        lp.chain_flags = d_chain_flags ? d_chain_flags + b0 : nullptr;
        if (use_sm) {
            bc::lu_sm_factor_kernel<<<cnt, bc::kLuSmThreads, bc::lu_sm_factor_smem(s), st>>>(lp);
            check_cuda(cudaGetLastError(), "lu_sm_factor_kernel launch");
            bc::lu_sm_solve_kernel<<<cnt, 32 * sm_warps, sm_solve_smem, st>>>(lp);
            check_cuda(cudaGetLastError(), "lu_sm_solve_kernel launch");
            ctx->launches += 2;
        } else {
            bc::lu_fallback_kernel<<<cnt, 256, smem, st>>>(lp);
            check_cuda(cudaGetLastError(), "lu_fallback_kernel launch");
            ctx->launches++;
        }
        ctx->kernels |= BC_KERNEL_LU;
    }
    std::vector<int32_t> status(ents.size());
    check_cuda(cudaMemcpyAsync(status.data(), ctx->lu_status.p, sizeof(int32_t) * ents.size(), cudaMemcpyDeviceToHost,
                               st), "D2H lu status");
    check_cuda(cudaStreamSynchronize(st), "lu_fallback_kernel");
    std::vector<bc::LuEntry> dense;
    for (size_t i = 0; i < ents.size(); ++i) {
        if (status[i] == 1) fail(BC_ERR_SINGULAR_MATRIX, "lu_solve: exactly singular matrix");
        if (status[i] == 2) dense.push_back(ents[i]);
    }
    if (!dense.empty()) {
        // one-cell groups reach status 2 only from the shared-memory kernels
        // (use_sm); the scratch kernel runs them densely already
        if (!blockdiag && !use_sm) fail(BC_ERR_CUDA, "lu_fallback_kernel: unexpected status");
        run_lu(ctx, dense, d_values, d_rhs, d_x, g_rms, s, nnz, block_width, st, 1);
    }
}

// The sign-of-zero chain (bc_lu.cuh, top) across the cells of one block-
// diagonal system solved cell by cell: cells run with no flips first; the scan
// redoes, in chain order, the few cells whose zeros an earlier (forward) or
// later (backward) cell flips, with the flags of their redone runs.
void lu_sign_chain(bc_ctx* ctx, int64_t cells, const double* d_values, const double* d_rhs, double* d_x, int s,
                   int nnz, uint8_t* d_fl, cudaStream_t st) {
    std::vector<uint8_t> fl(static_cast<size_t>(cells));
    check_cuda(cudaMemcpyAsync(fl.data(), d_fl, fl.size(), cudaMemcpyDeviceToHost, st), "D2H lu chain");
    check_cuda(cudaStreamSynchronize(st), "lu chain");
    std::vector<uint8_t> conv(fl.size(), 0), flip(fl.size(), 0);
    auto redo = [&](int64_t c, int later) {
        const std::vector<bc::LuEntry> one{{c, 0, 1, 0}};
        run_lu(ctx, one, d_values, d_rhs, d_x, nullptr, s, nnz, 0, st, 1, d_fl + c, conv[c], flip[c], later);
        check_cuda(cudaMemcpyAsync(&fl[c], d_fl + c, 1, cudaMemcpyDeviceToHost, st), "D2H lu chain");
        check_cuda(cudaStreamSynchronize(st), "lu chain");
    };
    bool neg_pivot = false, fwd = false;
    for (int64_t c = 0; c < cells; ++c) {
        conv[c] = neg_pivot && (fl[c] & bc::kChainNegZeroVal);
        flip[c] = fwd && (fl[c] & bc::kChainNegZeroRhs);
        if (conv[c] || flip[c]) redo(c, 0);
        neg_pivot = neg_pivot || (fl[c] & bc::kChainNegPivot);
        fwd = fwd || (fl[c] & bc::kChainFwd);
    }
    bool later = false;
    for (int64_t c = cells - 1; c >= 0; --c) {
        if (later && (fl[c] & bc::kChainNegZeroSum)) redo(c, 1);
        later = later || (fl[c] & bc::kChainBwd);
    }
}

struct MultiResult {
    int64_t iters = 0;
    double rms = 0.0;
    int32_t flags = 0;
};

// One cooperative launch of multi_cells_kernel over a global system of
// `cells` cells of pattern `pat` with the given reduction intervals.
MultiResult run_multi(bc_ctx* ctx, const bc::Pattern& pat, const int32_t* d_rp, const int32_t* d_ci,
                      const DevBuf& trp, const DevBuf& trow, const DevBuf& tval, const DevBuf& diag, int64_t cells,
                      const std::vector<int64_t>& ranges, const double* values, const double* rhs, const double* x0,
                      double* x, double tol, int64_t max_iter, int algo, int mode, cudaStream_t st) {
    const int64_t n = cells * pat.species, nb = static_cast<int64_t>(ranges.size() / 2);
    int64_t max_len = 1;
    for (int64_t b = 0; b < nb; ++b) max_len = std::max(max_len, ranges[2 * b + 1] - ranges[2 * b]);
    if (max_len > 4096) fail(BC_ERR_INVALID_ARGUMENT, "reduction interval longer than 4096 rows");
    check_cuda(ctx->m_ranges.ensure(sizeof(int64_t) * ranges.size()), "cudaMalloc(ranges)");
    check_cuda(cudaMemcpyAsync(ctx->m_ranges.p, ranges.data(), sizeof(int64_t) * ranges.size(),
                               cudaMemcpyHostToDevice, st), "H2D ranges");
    check_cuda(ctx->m_work.ensure(sizeof(double) * 7 * n), "cudaMalloc(multi work)");
    check_cuda(ctx->m_part.ensure(sizeof(double) * 2 * nb), "cudaMalloc(partials)");
    check_cuda(ctx->m_out.ensure(64), "cudaMalloc");
    bc::MultiParams p{};
    p.values = values;
    p.rhs = rhs;
    p.x0 = x0;
    p.x = x;
    p.row_ptr = d_rp;
    p.col_idx = d_ci;
    p.trow_ptr = trp.as<int32_t>();
    p.trow = trow.as<int32_t>();
    p.tval = tval.as<int32_t>();
    p.diag = diag.as<int32_t>();
    p.ranges = ctx->m_ranges.as<int64_t>();
    p.n_blocks = nb;
    p.n = n;
    p.species = pat.species;
    p.nnz = pat.nnz;
    p.max_len = static_cast<int>(max_len);
    p.work = ctx->m_work.as<double>();
    p.partials = ctx->m_part.as<double>();
    p.tol = tol;
    p.max_iter = max_iter;
    p.algo = algo == BC_ALGO_BICG ? bc::kBiCG : bc::kBiCGStab;
    p.mode = mode;
    p.out_iters = ctx->m_out.as<int64_t>();
    p.out_rms = reinterpret_cast<double*>(ctx->m_out.as<char>() + 8);
    p.out_flags = reinterpret_cast<int32_t*>(ctx->m_out.as<char>() + 16);
    int P2 = 256;
    while (P2 < max_len) P2 <<= 1;
    // two staging areas for the cells an interval's rows gather from (bc_multi.cuh mc_stage)
    const int64_t span = (max_len + 2 * static_cast<int64_t>(pat.species) - 2) / pat.species * pat.species;
    p.stage_len = 2 * span * 8 + 2 * P2 * 8 <= 160 * 1024 ? static_cast<int>(span) : 0;
    const size_t smem = sizeof(double) * (2 * P2 + 2 * static_cast<size_t>(p.stage_len));
    check_cuda(cudaFuncSetAttribute(bc::multi_cells_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)), "cudaFuncSetAttribute(multi)");
    int per_sm = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bc::multi_cells_kernel, 256, smem),
               "occupancy(multi)");
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(nb, static_cast<int64_t>(per_sm) * ctx->sms));
    void* args[] = {&p};
    check_cuda(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bc::multi_cells_kernel), dim3(grid), dim3(256),
                                           args, smem, st), "multi_cells_kernel cooperative launch");
    ctx->launches++;
    ctx->kernels |= BC_KERNEL_MULTI;
    MultiResult r;
    char buf[24];
    check_cuda(cudaMemcpyAsync(buf, ctx->m_out.p, 24, cudaMemcpyDeviceToHost, st), "D2H multi");
    check_cuda(cudaStreamSynchronize(st), "multi_cells_kernel");
    std::memcpy(&r.iters, buf, 8);
    std::memcpy(&r.rms, buf + 8, 8);
    std::memcpy(&r.flags, buf + 16, 4);
    return r;
}

extern "C" {

int bc_ctx_create(int device, bc_ctx** out) {
    if (!out) return BC_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    bc_ctx* ctx = new (std::nothrow) bc_ctx;
    if (!ctx) return BC_ERR_NO_MEMORY;
    ctx->device = device;
    const int st = guarded(ctx, [&] {
        check_cuda(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device),
                   "cudaDeviceGetAttribute");
        int major = 0;
        check_cuda(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device),
                   "cudaDeviceGetAttribute");
        if (major != 10) fail(BC_ERR_CUDA, "libbc_b200 is built for sm_100a (B200) only");
        check_cuda(cudaEventCreate(&ctx->e0), "cudaEventCreate");
        check_cuda(cudaEventCreate(&ctx->e1), "cudaEventCreate");
        check_cuda(ctx->counters.ensure(64 * sizeof(unsigned int)), "cudaMalloc");
        check_cuda(cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking), "cudaStreamCreate");
        for (cudaEvent_t& e : ctx->pipe_ev)
            check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        check_cuda(ctx->pipe_flags.ensure(sizeof(unsigned int) * (kPipeFlags + 1)), "cudaMalloc(flags)");
        check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_ones), sizeof(unsigned int), cudaHostAllocDefault),
                   "cudaHostAlloc");
        ctx->h_ones[0] = 1u;
        return BC_OK;
    });
    if (st != BC_OK) {
        std::fprintf(stderr, "bc_ctx_create: %s\n", ctx->err.c_str());
        delete ctx;
        return st;
    }
    *out = ctx;
    return BC_OK;
}

void bc_ctx_destroy(bc_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (DevBuf* b : {&ctx->d_rp, &ctx->d_ci, &ctx->values, &ctx->rhs, &ctx->x, &ctx->giters,
                      &ctx->grms, &ctx->gflags, &ctx->counters, &ctx->lu_scratch,
                      &ctx->lu_entries, &ctx->lu_status, &ctx->f_scratch, &ctx->lu_rms_scratch, &ctx->lu_chain, &ctx->t_values,
                      &ctx->t_work, &ctx->m_trp, &ctx->m_trow, &ctx->m_tval, &ctx->m_diag, &ctx->m_ranges,
                      &ctx->m_work, &ctx->m_part, &ctx->m_out, &ctx->sim_tabs, &ctx->sim_sign, &ctx->sim_rates,
                      &ctx->sim_y, &ctx->sim_prev, &ctx->sim_values, &ctx->sim_rhs, &ctx->sim_dx, &ctx->sim_red})
        b->release();
    for (DevBuf& b : ctx->plan_bufs) b.release();
    if (ctx->e0) cudaEventDestroy(ctx->e0);
    if (ctx->e1) cudaEventDestroy(ctx->e1);
    for (cudaEvent_t e : ctx->pipe_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_st) cudaStreamDestroy(ctx->copy_st);
    ctx->pipe_flags.release();
    if (ctx->h_ones) cudaFreeHost(ctx->h_ones);
    delete ctx;
}

const char* bc_last_error(const bc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int64_t bc_kernel_launches(const bc_ctx* ctx) { return ctx ? ctx->launches : 0; }

int bc_set_pattern(bc_ctx* ctx, int32_t species, const int32_t* row_ptr, const int32_t* col_idx) {
    if (!ctx) return BC_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        bc::Pattern p = make_pattern(species, row_ptr, col_idx);
        // Same pattern as installed: keep its schedules.  The comparison is
        // against the context's own state, so a pattern installed behind a
        // caller's back (bc_simulate installs the mechanism's) is never reused
        // by mistake.
        if (ctx->has_pattern && p.species == ctx->pat.species && p.row_ptr == ctx->pat.row_ptr &&
            p.col_idx == ctx->pat.col_idx)
            return BC_OK;
        ctx->plans.clear();
        ctx->lat_plans.clear();
        for (DevBuf& b : ctx->plan_bufs) b.release();
        ctx->plan_bufs.clear();
        check_cuda(ctx->d_rp.ensure(sizeof(int32_t) * p.row_ptr.size()), "cudaMalloc");
        check_cuda(ctx->d_ci.ensure(sizeof(int32_t) * std::max<size_t>(p.col_idx.size(), 1)), "cudaMalloc");
        check_cuda(cudaMemcpy(ctx->d_rp.p, p.row_ptr.data(), sizeof(int32_t) * p.row_ptr.size(),
                              cudaMemcpyHostToDevice), "cudaMemcpy");
        if (!p.col_idx.empty())
            check_cuda(cudaMemcpy(ctx->d_ci.p, p.col_idx.data(), sizeof(int32_t) * p.col_idx.size(),
                                  cudaMemcpyHostToDevice), "cudaMemcpy");
        ctx->pat = std::move(p);
        ctx->m_ready = false;
        ctx->has_pattern = true;
        return BC_OK;
    });
}

int bc_ctx_pattern_info(const bc_ctx* ctx, int32_t* info) {
    if (!ctx || !info) return BC_ERR_INVALID_ARGUMENT;
    if (!ctx->has_pattern) return BC_ERR_NO_PATTERN;
    info[0] = ctx->pat.species;
    info[1] = ctx->pat.nnz;
    return BC_OK;
}

int bc_plan(int32_t species, const bc_solve_params* prm, int64_t* n_groups, double* cpb) {
    if (!prm || !n_groups || !cpb) return BC_ERR_INVALID_ARGUMENT;
    return guarded(nullptr, [&] {
        if (species < 1) fail(BC_ERR_INVALID_ARGUMENT, "batched system: no species");
        plan_groups(prm, species, cpb, n_groups, nullptr);
        return BC_OK;
    });
}

int bc_schedule_export(int32_t species, const int32_t* row_ptr, const int32_t* col_idx, int32_t k,
                       int32_t with_t, int32_t* info, uint32_t* words, int32_t* vpos, int32_t* xpos,
                       uint32_t* twords, int32_t* tvpos, int32_t* txpos) {
    if (!info || k < 1) return BC_ERR_INVALID_ARGUMENT;
    return guarded(nullptr, [&] {
        const bc::Pattern pat = make_pattern(species, row_ptr, col_idx);
        const bc::GroupPlan gp = bc::build_group_plan(pat, k, with_t != 0);
        const int v[12] = {gp.geo.n, gp.geo.P, gp.geo.Q, gp.geo.W, gp.geo.R, gp.geo.RV, gp.a.steps,
                           with_t ? gp.at.steps : 0, gp.a.xslots, with_t ? gp.at.xslots : 0,
                           gp.a.conflict_cost, with_t ? gp.at.conflict_cost : 0};
        std::memcpy(info, v, sizeof v);
        if (words) std::memcpy(words, gp.a.words.data(), sizeof(uint32_t) * gp.a.words.size());
        if (vpos) std::memcpy(vpos, gp.a.vpos.data(), sizeof(int32_t) * gp.a.vpos.size());
        if (xpos) std::memcpy(xpos, gp.a.xpos.data(), sizeof(int32_t) * gp.a.xpos.size());
        if (with_t && txpos) std::memcpy(txpos, gp.at.xpos.data(), sizeof(int32_t) * gp.at.xpos.size());
        if (with_t && twords) std::memcpy(twords, gp.at.words.data(), sizeof(uint32_t) * gp.at.words.size());
        if (with_t && tvpos) std::memcpy(tvpos, gp.at.vpos.data(), sizeof(int32_t) * gp.at.vpos.size());
        return BC_OK;
    });
}

int bc_tmem_schedule_export(int32_t species, const int32_t* row_ptr, const int32_t* col_idx, int32_t k,
                            int32_t pair, int32_t team, int32_t* info, uint16_t* words, int32_t* vidx,
                            int32_t* xpos, int32_t* yslot) {
    if (!info || k < 1) return BC_ERR_INVALID_ARGUMENT;
    return guarded(nullptr, [&] {
        const bc::Pattern pat = make_pattern(species, row_ptr, col_idx);
        if (team != 1 && team != 2 && team != 4) fail(BC_ERR_INVALID_ARGUMENT, "team must be 1, 2 or 4");
        const bc::TmemSchedule ts = bc::build_tmem_schedule(pat, k, pair != 0, team);
        const int v[9] = {ts.steps,  ts.xslots,      ts.zero_slot, ts.yslots, ts.conflict_cost,
                          ts.copies, ts.model_total, ts.streams,   ts.ystream};
        std::memcpy(info, v, sizeof v);
        if (words) std::memcpy(words, ts.words.data(), sizeof(uint16_t) * ts.words.size());
        if (vidx) std::memcpy(vidx, ts.vidx.data(), sizeof(int32_t) * ts.vidx.size());
        if (xpos) std::memcpy(xpos, ts.xpos.data(), sizeof(int32_t) * ts.xpos.size());
        if (yslot) std::memcpy(yslot, ts.yslot.data(), sizeof(int32_t) * ts.yslot.size());
        return BC_OK;
    });
}

int bc_latency_schedule_export(int32_t species, const int32_t* row_ptr, const int32_t* col_idx, int32_t k,
                               int32_t bicg, int32_t threads, int32_t* info, int32_t* rowof, int32_t* steps,
                               int32_t* rvi, uint16_t* rxo, int32_t* tvi, uint16_t* txo, int32_t* didx) {
    if (!info || k < 1) return BC_ERR_INVALID_ARGUMENT;
    return guarded(nullptr, [&] {
        const bc::Pattern pat = make_pattern(species, row_ptr, col_idx);
        const bc::LatencySchedule ls = bc::build_latency_schedule(pat, k, bicg != 0, threads);
        const int v[8] = {ls.n, ls.P, ls.T, ls.lmax, ls.L, ls.xslots, ls.model_wavefronts, ls.lmax <= 32 ? 1 : 0};
        std::memcpy(info, v, sizeof v);
        if (ls.lmax > 32) return BC_OK;  // no tables: the kernel has no instance for it
        if (rowof) std::memcpy(rowof, ls.rowof.data(), sizeof(int32_t) * ls.rowof.size());
        if (steps) std::memcpy(steps, ls.steps.data(), sizeof(int32_t) * ls.steps.size());
        if (rvi) std::memcpy(rvi, ls.rvi.data(), sizeof(int32_t) * ls.rvi.size());
        if (rxo) std::memcpy(rxo, ls.rxo.data(), sizeof(uint16_t) * ls.rxo.size());
        if (bicg && tvi) std::memcpy(tvi, ls.tvi.data(), sizeof(int32_t) * ls.tvi.size());
        if (bicg && txo) std::memcpy(txo, ls.txo.data(), sizeof(uint16_t) * ls.txo.size());
        if (didx) std::memcpy(didx, ls.didx.data(), sizeof(int32_t) * ls.didx.size());
        return BC_OK;
    });
}

int bc_solve(bc_ctx* ctx, const bc_solve_params* prm, const double* values, const double* rhs,
             double* x_out, int32_t* group_iters, double* group_rms, uint8_t* group_flags,
             bc_report* report) {
    if (!ctx || !prm) return BC_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&]() -> int {
        if (!ctx->has_pattern) fail(BC_ERR_NO_PATTERN, "bc_set_pattern has not been called");
        const bc::Pattern& pat = ctx->pat;
        if (!values || !rhs || !x_out) fail(BC_ERR_INVALID_ARGUMENT, "null values/rhs/x_out");
        double cpb = 0.0;
        int64_t n_groups = 0;
        std::vector<GroupSpan> spans;
        plan_groups(prm, pat.species, &cpb, &n_groups, &spans);
        if (!(prm->tol > 0.0)) fail(BC_ERR_INVALID_ARGUMENT, "bicg: tol must be positive");
        if (prm->max_iter < 1) fail(BC_ERR_INVALID_ARGUMENT, "bicg: max_iter must be >= 1");
        if (prm->algo != BC_ALGO_BICG && prm->algo != BC_ALGO_BICGSTAB_JACOBI)
            fail(BC_ERR_INVALID_ARGUMENT, "unknown algorithm");

        cudaStream_t st = static_cast<cudaStream_t>(prm->stream);
        const int64_t cells = prm->cells, s = pat.species, nnz = pat.nnz;
        const size_t vbytes = sizeof(double) * cells * nnz, bbytes = sizeof(double) * cells * s;
        const double* d_values = values;
        const double* d_rhs = rhs;
        double* d_x = x_out;
        // Host inputs of a Block-cells / One-cell solve stream in by chunks while
        // the kernel runs: every chunk's copy is queued on copy_st BEFORE the
        // launch, followed by its ready flag; the kernel's warps wait for the
        // flag of their group's chunk (InputGate).  Queued first, the copies
        // also complete first wherever work is serialised (profilers,
        // CUDA_LAUNCH_BLOCKING), so the gate can never wait on later work.
        const bool pipelined = !is_device_ptr(values) && !is_device_ptr(rhs) &&
                               prm->strategy != BC_STRATEGY_MULTI_CELLS &&
                               prm->strategy != BC_STRATEGY_THREAD_PER_CELL && cells >= kPipeMinCells &&
                               std::getenv("BC_NO_PIPELINE") == nullptr;
        if (pipelined) {
            check_cuda(ctx->values.ensure(vbytes), "cudaMalloc(values)");
            check_cuda(ctx->rhs.ensure(bbytes), "cudaMalloc(rhs)");
            d_values = ctx->values.as<double>();
            d_rhs = ctx->rhs.as<double>();
        } else if (!is_device_ptr(values)) {
            check_cuda(ctx->values.ensure(vbytes), "cudaMalloc(values)");
            check_cuda(cudaMemcpyAsync(ctx->values.p, values, vbytes, cudaMemcpyHostToDevice, st), "H2D values");
            d_values = ctx->values.as<double>();
        }
        if (!pipelined && !is_device_ptr(rhs)) {
            check_cuda(ctx->rhs.ensure(bbytes), "cudaMalloc(rhs)");
            check_cuda(cudaMemcpyAsync(ctx->rhs.p, rhs, bbytes, cudaMemcpyHostToDevice, st), "H2D rhs");
            d_rhs = ctx->rhs.as<double>();
        }
        bool host_x = !is_device_ptr(x_out);
        if (host_x && pipelined) {  // pinned x_out: the kernels write the solution straight to host memory
            if (double* mapped = static_cast<double*>(mapped_host_ptr(x_out))) {
                d_x = mapped;
                host_x = false;
            }
        }
        if (host_x) {
            check_cuda(ctx->x.ensure(bbytes), "cudaMalloc(x)");
            d_x = ctx->x.as<double>();
        }
        check_cuda(ctx->giters.ensure(sizeof(int32_t) * n_groups), "cudaMalloc");
        check_cuda(ctx->grms.ensure(sizeof(double) * n_groups), "cudaMalloc");
        check_cuda(ctx->gflags.ensure(n_groups), "cudaMalloc");
        const int64_t launches0 = ctx->launches;
        ctx->kernels = 0;

        const bool timing = (prm->options & BC_OPT_TIMING) != 0;
        const bool bicg = prm->algo == BC_ALGO_BICG;
        const bool multi = prm->strategy == BC_STRATEGY_MULTI_CELLS;
        const bool tpc = prm->strategy == BC_STRATEGY_THREAD_PER_CELL;
        const int64_t mtpb = prm->max_threads_per_block > 0 ? prm->max_threads_per_block : 1024;
        std::vector<int64_t> multi_ranges;
        if (multi) {  // exec_model.cpp:202-220: one interval per 1024-thread block + host stage
            spans[0].k = static_cast<int>(prm->cells);
            if (!ctx->m_ready) {
                upload_multi_tables(pat, &ctx->m_trp, &ctx->m_trow, &ctx->m_tval, &ctx->m_diag);
                ctx->m_ready = true;
            }
            const int64_t ntot = prm->cells * s;
            for (int64_t b0 = 0; b0 < ntot; b0 += mtpb) {
                multi_ranges.push_back(b0);
                multi_ranges.push_back(std::min(ntot, b0 + mtpb));
            }
        } else if (tpc) {
            if (!ctx->m_ready) {
                upload_multi_tables(pat, &ctx->m_trp, &ctx->m_trow, &ctx->m_tval, &ctx->m_diag);
                ctx->m_ready = true;
            }
            check_cuda(ctx->t_values.ensure(sizeof(double) * prm->cells * nnz), "cudaMalloc(interleaved)");
            check_cuda(ctx->t_work.ensure(sizeof(double) * 9 * prm->cells * s), "cudaMalloc(thread work)");
        } else {
            for (const GroupSpan& sp : spans) {  // host-side planning before the timed region
                bc::GroupPlan& gp = get_plan(ctx, pat, sp.k, bicg, &ctx->plans);
                if (latency_wanted(ctx, sp.count) && latency_plan(ctx, pat, sp.k, bicg).ok) continue;
                const TmemCfg* cfg = nullptr;
                if (bc::TmemPlan* tp = tmem_plan(ctx, pat, gp, sp.count, &cfg))
                    ensure_tmem_lane_tables(ctx, gp, *tp, cfg->RV);
            }
        }
        if (timing) check_cuda(cudaEventRecord(ctx->e0, st), "cudaEventRecord");
        int slot = 0;
        if (multi) {
            const MultiResult mr = run_multi(ctx, pat, ctx->d_rp.as<int32_t>(), ctx->d_ci.as<int32_t>(), ctx->m_trp,
                                             ctx->m_trow, ctx->m_tval, ctx->m_diag, prm->cells, multi_ranges,
                                             d_values, d_rhs, nullptr, d_x, prm->tol, prm->max_iter, prm->algo, 0, st);
            const int32_t it32 = static_cast<int32_t>(mr.iters);
            const uint8_t f8 = static_cast<uint8_t>(mr.flags);
            check_cuda(cudaMemcpyAsync(ctx->giters.p, &it32, 4, cudaMemcpyHostToDevice, st), "H2D");
            check_cuda(cudaMemcpyAsync(ctx->grms.p, &mr.rms, 8, cudaMemcpyHostToDevice, st), "H2D");
            check_cuda(cudaMemcpyAsync(ctx->gflags.p, &f8, 1, cudaMemcpyHostToDevice, st), "H2D");
            check_cuda(cudaStreamSynchronize(st), "H2D multi outputs");
        }
        if (tpc) {  // one thread per cell (bc_thread.cuh)
            const dim3 tb(32, 8), tg(static_cast<unsigned>((prm->cells + 31) / 32), static_cast<unsigned>((nnz + 31) / 32));
            bc::interleave_kernel<<<tg, tb, 0, st>>>(d_values, ctx->t_values.as<double>(), prm->cells,
                                                     static_cast<int>(nnz));
            check_cuda(cudaGetLastError(), "interleave_kernel launch");
            bc::ThreadParams tp{};
            tp.values_il = ctx->t_values.as<double>();
            tp.rhs = d_rhs;
            tp.x_out = d_x;
            tp.work = ctx->t_work.as<double>();
            tp.row_ptr = ctx->d_rp.as<int32_t>();
            tp.col_idx = ctx->d_ci.as<int32_t>();
            tp.diag = ctx->m_diag.as<int32_t>();
            tp.g_iters = ctx->giters.as<int32_t>();
            tp.g_rms = ctx->grms.as<double>();
            tp.g_flags = ctx->gflags.as<uint8_t>();
            tp.cells = prm->cells;
            tp.species = static_cast<int>(s);
            tp.nnz = static_cast<int>(nnz);
            int lg = 0;
            while ((int64_t(1) << lg) < s) ++lg;
            tp.log2P = lg;
            tp.tol = prm->tol;
            tp.max_iter = prm->max_iter;
            const unsigned blocks = static_cast<unsigned>((prm->cells + 127) / 128);
            if (bicg)
                bc::thread_per_cell_kernel<bc::kBiCG><<<blocks, 128, 0, st>>>(tp);
            else
                bc::thread_per_cell_kernel<bc::kBiCGStab><<<blocks, 128, 0, st>>>(tp);
            check_cuda(cudaGetLastError(), "thread_per_cell_kernel launch");
            ctx->launches += 2;
            ctx->kernels |= BC_KERNEL_THREAD;
        }
        // streamed inputs: chunks of each span, each a whole number of 128-byte
        // lines of values and rhs; all copies and flags queued before the launches
        std::vector<bc::InputGate> gates(spans.size(), bc::InputGate{nullptr, nullptr, 1, 0});
        if (pipelined) {
            unsigned int* flags_d = ctx->pipe_flags.as<unsigned int>();
            check_cuda(cudaMemsetAsync(flags_d, 0, sizeof(unsigned int) * (kPipeFlags + 1), st), "memset flags");
            check_cuda(cudaEventRecord(ctx->pipe_ev[0], st), "cudaEventRecord");
            check_cuda(cudaStreamWaitEvent(ctx->copy_st, ctx->pipe_ev[0]), "cudaStreamWaitEvent");
            int base = 0;
            for (size_t i = 0; i < spans.size(); ++i) {
                const GroupSpan& sp = spans[i];
                const int align = 16 / std::gcd(16, sp.k);
                int per = std::max(align, (sp.count + pipe_chunks() - 1) / pipe_chunks());
                per = (per + align - 1) / align * align;
                gates[i] = bc::InputGate{flags_d, flags_d + kPipeFlags, per, base};
                for (int g0 = 0; g0 < sp.count; g0 += per, ++base) {
                    const int64_t c0 = sp.cell0 + static_cast<int64_t>(g0) * sp.k;
                    const int64_t nc = static_cast<int64_t>(std::min(per, sp.count - g0)) * sp.k;
                    check_cuda(cudaMemcpyAsync(ctx->values.as<double>() + c0 * nnz, values + c0 * nnz,
                                               sizeof(double) * nc * nnz, cudaMemcpyHostToDevice, ctx->copy_st),
                               "H2D values chunk");
                    check_cuda(cudaMemcpyAsync(ctx->rhs.as<double>() + c0 * s, rhs + c0 * s, sizeof(double) * nc * s,
                                               cudaMemcpyHostToDevice, ctx->copy_st), "H2D rhs chunk");
                    check_cuda(cudaMemcpyAsync(flags_d + base, ctx->h_ones, sizeof(unsigned int),
                                               cudaMemcpyHostToDevice, ctx->copy_st), "H2D ready flag");
                }
            }
            if (base > kPipeFlags) fail(BC_ERR_INVALID_ARGUMENT, "input pipeline: too many chunks");
            check_cuda(cudaEventRecord(ctx->pipe_ev[1], ctx->copy_st), "cudaEventRecord");
        }
        for (size_t i = 0; i < spans.size(); ++i) {
            if (multi || tpc) break;
            const GroupSpan& sp = spans[i];
            bc::GroupPlan& gp = get_plan(ctx, pat, sp.k, bicg, &ctx->plans);
            unsigned int* counter = ctx->counters.as<unsigned int>() + slot++;
            if (launch_latency(ctx, pat, gp, prm->algo, sp.cell0, sp.gout0, sp.count, d_values, d_rhs, d_x,
                               prm->tol, prm->max_iter, st, gates[i]))
                continue;
            if (!launch_tmem(ctx, pat, gp, sp.cell0, sp.gout0, sp.count, d_values, d_rhs, d_x, prm->tol,
                                     prm->max_iter, counter, st, gates[i]))
                launch_block(ctx, pat, gp, prm->algo, sp.cell0, sp.gout0, sp.count, d_values, d_rhs, nullptr, d_x,
                             prm->tol, prm->max_iter, counter, st, gates[i]);
        }
        if (pipelined) check_cuda(cudaStreamWaitEvent(st, ctx->pipe_ev[1]), "cudaStreamWaitEvent");  // join
        // breakdown groups -> device LU fallback
        std::vector<uint8_t> flags(n_groups);
        check_cuda(cudaMemcpyAsync(flags.data(), ctx->gflags.p, n_groups, cudaMemcpyDeviceToHost, st), "D2H flags");
        unsigned int gate_err = 0;
        if (pipelined)
            check_cuda(cudaMemcpyAsync(&gate_err, ctx->pipe_flags.as<unsigned int>() + kPipeFlags, sizeof gate_err,
                                       cudaMemcpyDeviceToHost, st), "D2H gate error");
        check_cuda(cudaStreamSynchronize(st), "solve kernels");
        if (gate_err) fail(BC_ERR_CUDA, "input pipeline: a chunk of the host inputs never arrived");
        std::vector<bc::LuEntry> ents;
        for (const GroupSpan& sp : spans)
            for (int g = 0; g < sp.count; ++g) {
                const int64_t go = sp.gout0 + g;
                if (flags[go] & BC_FLAG_BREAKDOWN)
                    ents.push_back({sp.cell0 + static_cast<int64_t>(g) * sp.k, go, sp.k, 0});
            }
        int64_t fallbacks = 0;
        if (!ents.empty()) {
            const int64_t ntot = prm->cells * s;
            if (multi && ntot > 2048) {
                // Multi-cells breakdown on a large system: the block-diagonal
                // LU runs cell by cell, and the host replays the chain of
                // sign-of-zero rules the reference's dense LU (strategies.cpp:47)
                // applies across cells (bc_lu.cuh), then the fallback residual
                // goes through the global plan.
                std::vector<bc::LuEntry> cells_e;
                for (int64_t c = 0; c < prm->cells; ++c) cells_e.push_back({c, 0, 1, 0});
                check_cuda(ctx->lu_rms_scratch.ensure(sizeof(double) * 8), "cudaMalloc");
                check_cuda(ctx->lu_chain.ensure(static_cast<size_t>(prm->cells)), "cudaMalloc(lu chain)");
                uint8_t* d_fl = ctx->lu_chain.as<uint8_t>();
                run_lu(ctx, cells_e, d_values, d_rhs, d_x, nullptr, static_cast<int>(s), static_cast<int>(nnz), 0, st,
                       1, d_fl);
                lu_sign_chain(ctx, prm->cells, d_values, d_rhs, d_x, static_cast<int>(s), static_cast<int>(nnz), d_fl,
                              st);
                const MultiResult mr = run_multi(ctx, pat, ctx->d_rp.as<int32_t>(), ctx->d_ci.as<int32_t>(), ctx->m_trp,
                                                 ctx->m_trow, ctx->m_tval, ctx->m_diag, prm->cells, multi_ranges,
                                                 d_values, d_rhs, nullptr, d_x, prm->tol, prm->max_iter, prm->algo,
                                                 1, st);
                check_cuda(cudaMemcpyAsync(ctx->grms.p, &mr.rms, sizeof(double), cudaMemcpyHostToDevice, st),
                           "H2D rms");
            } else {
                run_lu(ctx, ents, d_values, d_rhs, d_x, ctx->grms.as<double>(), static_cast<int>(s),
                       static_cast<int>(nnz), multi ? static_cast<int>(mtpb) : 0, st);
            }
            for (const auto& e : ents) flags[e.gout] |= BC_FLAG_FELL_BACK;
            fallbacks = static_cast<int64_t>(ents.size());
        }
        if (timing) check_cuda(cudaEventRecord(ctx->e1, st), "cudaEventRecord");

        // outputs
        if (host_x)
            check_cuda(cudaMemcpyAsync(x_out, d_x, bbytes, cudaMemcpyDeviceToHost, st), "D2H x");
        std::vector<int32_t> h_it;
        std::vector<double> h_rms;
        int32_t* it_dst = group_iters;
        double* rms_dst = group_rms;
        const bool it_dev = is_device_ptr(group_iters), rms_dev = is_device_ptr(group_rms);
        h_it.resize(n_groups);
        h_rms.resize(n_groups);
        check_cuda(cudaMemcpyAsync(h_it.data(), ctx->giters.p, sizeof(int32_t) * n_groups,
                                   cudaMemcpyDeviceToHost, st), "D2H iters");
        check_cuda(cudaMemcpyAsync(h_rms.data(), ctx->grms.p, sizeof(double) * n_groups,
                                   cudaMemcpyDeviceToHost, st), "D2H rms");
        if (it_dst && it_dev)
            check_cuda(cudaMemcpyAsync(it_dst, ctx->giters.p, sizeof(int32_t) * n_groups,
                                       cudaMemcpyDeviceToDevice, st), "D2D iters");
        if (rms_dst && rms_dev)
            check_cuda(cudaMemcpyAsync(rms_dst, ctx->grms.p, sizeof(double) * n_groups,
                                       cudaMemcpyDeviceToDevice, st), "D2D rms");
        if (group_flags && is_device_ptr(group_flags))
            check_cuda(cudaMemcpyAsync(group_flags, flags.data(), n_groups, cudaMemcpyHostToDevice, st),
                       "H2D flags");
        check_cuda(cudaStreamSynchronize(st), "outputs");
        if (it_dst && !it_dev) std::memcpy(it_dst, h_it.data(), sizeof(int32_t) * n_groups);
        if (rms_dst && !rms_dev) std::memcpy(rms_dst, h_rms.data(), sizeof(double) * n_groups);
        if (group_flags && !is_device_ptr(group_flags)) std::memcpy(group_flags, flags.data(), n_groups);

        if (report) {  // merge_groups, strategies.cpp:71-87
            std::memset(report, 0, sizeof *report);
            report->n_groups = n_groups;
            report->cells_per_block = cpb;
            for (int64_t g = 0; g < n_groups; ++g) {
                report->iterations_sum += h_it[g];
                report->iterations_effective = std::max<int64_t>(report->iterations_effective, h_it[g]);
                if (h_rms[g] > report->max_residual_rms) report->max_residual_rms = h_rms[g];
            }
            report->breakdown_fallbacks = fallbacks;
            report->kernel_launches = ctx->launches - launches0;
            report->kernels = ctx->kernels;
            report->model_spmv_wavefronts = (ctx->kernels & BC_KERNEL_TMEM) ? ctx->model_spmv_wf : 0.0;
            if (timing) {
                float ms = 0.f;
                check_cuda(cudaEventElapsedTime(&ms, ctx->e0, ctx->e1), "cudaEventElapsedTime");
                report->device_ms = ms;
            }
        }
        return BC_OK;
    });
}

int bc_bicg_solve(bc_ctx* ctx, int32_t algo, int32_t n, const int32_t* row_ptr, const int32_t* col_idx,
                  const double* vals, const double* b, const double* x0, double tol, int64_t max_iter,
                  int64_t n_blocks, const int64_t* ranges, double* x_out, bc_outcome* out) {
    if (!ctx) return BC_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&]() -> int {
        if (n < 1) fail(BC_ERR_INVALID_ARGUMENT, "bicg: matrix not square / empty");
        if (!vals || !b || !x_out || !out) fail(BC_ERR_INVALID_ARGUMENT, "bicg: null pointer");
        if (!(tol > 0.0)) fail(BC_ERR_INVALID_ARGUMENT, "bicg: tol must be positive");
        if (max_iter < 1) fail(BC_ERR_INVALID_ARGUMENT, "bicg: max_iter must be >= 1");
        if (algo != BC_ALGO_BICG && algo != BC_ALGO_BICGSTAB_JACOBI)
            fail(BC_ERR_INVALID_ARGUMENT, "unknown algorithm");
        // reduction.cpp:16-25 check_partition
        int64_t expect = 0;
        for (int64_t k = 0; k < n_blocks; ++k) {
            if (ranges[2 * k] != expect || ranges[2 * k + 1] <= ranges[2 * k])
                fail(BC_ERR_INVALID_ARGUMENT, "reduction plan does not partition [0, n)");
            expect = ranges[2 * k + 1];
        }
        if (expect != n) fail(BC_ERR_INVALID_ARGUMENT, "reduction plan does not cover [0, n)");
        const bc::Pattern pat = make_pattern(n, row_ptr, col_idx);
        if (n_blocks != 1 || n > bc::kMaxGroupRows) {
            // general ReductionPlan (several intervals + sequential combine):
            // the Multi-cells kernel over one "cell" holding the whole system
            DevBuf rp, ci, trp, trow, tval, dg, dv, db, dx0, dx;
            auto up = [](DevBuf* b, const void* src, size_t bytes) {
                check_cuda(b->ensure(std::max<size_t>(bytes, 8)), "cudaMalloc");
                if (bytes) check_cuda(cudaMemcpy(b->p, src, bytes, cudaMemcpyDefault), "copy");
            };
            up(&rp, pat.row_ptr.data(), sizeof(int32_t) * pat.row_ptr.size());
            up(&ci, pat.col_idx.data(), sizeof(int32_t) * pat.col_idx.size());
            up(&dv, vals, sizeof(double) * pat.nnz);
            up(&db, b, sizeof(double) * n);
            if (x0) up(&dx0, x0, sizeof(double) * n);
            check_cuda(dx.ensure(sizeof(double) * n), "cudaMalloc");
            upload_multi_tables(pat, &trp, &trow, &tval, &dg);
            std::vector<int64_t> rg(ranges, ranges + 2 * n_blocks);
            const MultiResult mr = run_multi(ctx, pat, rp.as<int32_t>(), ci.as<int32_t>(), trp, trow, tval, dg, 1, rg,
                                             dv.as<double>(), db.as<double>(), x0 ? dx0.as<double>() : nullptr,
                                             dx.as<double>(), tol, max_iter, algo, 0, 0);
            check_cuda(cudaMemcpy(x_out, dx.p, sizeof(double) * n, cudaMemcpyDefault), "copy x");
            for (DevBuf* d : {&rp, &ci, &trp, &trow, &tval, &dg, &dv, &db, &dx0, &dx}) d->release();
            out->iterations = mr.iters;
            out->final_residual_rms = mr.rms;
            out->converged = (mr.flags & BC_FLAG_CONVERGED) ? 1 : 0;
            out->breakdown = (mr.flags & BC_FLAG_BREAKDOWN) ? 1 : 0;
            return BC_OK;
        }
        std::map<std::pair<int, int>, bc::GroupPlan> local;
        const size_t first_buf = ctx->plan_bufs.size();
        const bc::GroupPlan& gp = get_plan(ctx, pat, 1, algo == BC_ALGO_BICG, &local);
        const size_t vb = sizeof(double) * pat.nnz, bb = sizeof(double) * n;
        check_cuda(ctx->values.ensure(std::max<size_t>(vb, 8)), "cudaMalloc");
        check_cuda(ctx->rhs.ensure(bb * 2), "cudaMalloc");
        check_cuda(ctx->x.ensure(bb), "cudaMalloc");
        check_cuda(ctx->giters.ensure(4), "cudaMalloc");
        check_cuda(ctx->grms.ensure(8), "cudaMalloc");
        check_cuda(ctx->gflags.ensure(1), "cudaMalloc");
        const cudaMemcpyKind kin = cudaMemcpyDefault;
        if (vb) check_cuda(cudaMemcpy(ctx->values.p, vals, vb, kin), "copy values");
        check_cuda(cudaMemcpy(ctx->rhs.p, b, bb, kin), "copy b");
        double* d_x0 = nullptr;
        if (x0) {
            d_x0 = ctx->rhs.as<double>() + n;
            check_cuda(cudaMemcpy(d_x0, x0, bb, kin), "copy x0");
        }
        launch_block(ctx, pat, gp, algo, 0, 0, 1, ctx->values.as<double>(), ctx->rhs.as<double>(), d_x0,
                     ctx->x.as<double>(), tol, max_iter, ctx->counters.as<unsigned int>() + 8, 0);
        check_cuda(cudaDeviceSynchronize(), "bicg kernel");
        int32_t it = 0;
        double rms = 0.0;
        uint8_t fl = 0;
        check_cuda(cudaMemcpy(x_out, ctx->x.p, bb, kin), "copy x");
        check_cuda(cudaMemcpy(&it, ctx->giters.p, 4, cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(&rms, ctx->grms.p, 8, cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(&fl, ctx->gflags.p, 1, cudaMemcpyDeviceToHost), "D2H");
        for (size_t i = first_buf; i < ctx->plan_bufs.size(); ++i) ctx->plan_bufs[i].release();
        ctx->plan_bufs.resize(first_buf);
        out->iterations = it;
        out->final_residual_rms = rms;
        out->converged = (fl & BC_FLAG_CONVERGED) ? 1 : 0;
        out->breakdown = (fl & BC_FLAG_BREAKDOWN) ? 1 : 0;
        return BC_OK;
    });
}

int bc_newton_assemble(bc_ctx* ctx, int64_t count, int32_t species, int32_t reactions, int32_t nnz,
                       const double* rates, const int32_t* stamp_ptr, const int32_t* stamp_slot,
                       const double* stamp_sign, const int32_t* stamp_other, const int32_t* reactant_ptr,
                       const int32_t* reactants, const int32_t* product_ptr, const int32_t* products,
                       const int32_t* diag_slot, double h, const double* y, const double* y_prev,
                       double* values, double* rhs, void* stream) {
    if (!ctx) return BC_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&]() -> int {
        if (count < 0 || species < 1 || reactions < 1 || nnz < 1 || !(h > 0.0))
            fail(BC_ERR_INVALID_ARGUMENT, "newton_assemble: bad sizes");
        if (count == 0) return BC_OK;
        check_cuda(ctx->f_scratch.ensure(sizeof(double) * count * species), "cudaMalloc");
        bc::NewtonParams p{count, species, reactions, nnz, rates, stamp_ptr, stamp_slot, stamp_other,
                           stamp_sign, reactant_ptr, reactants, product_ptr, products, diag_slot,
                           h, y, y_prev, values, rhs, ctx->f_scratch.as<double>()};
        const int threads = 128;
        const int64_t blocks = (count + threads - 1) / threads;
        bc::newton_assemble_kernel<<<static_cast<unsigned>(blocks), threads, 0,
                                     static_cast<cudaStream_t>(stream)>>>(p);
        check_cuda(cudaGetLastError(), "newton_assemble_kernel launch");
        ctx->launches++;
        return BC_OK;
    });
}

int bc_simulate(bc_ctx* ctx, const bc_sim_params* prm, const bc_mechanism_tables* mt, const double* rates,
                double* states, bc_step_stats* per_step, int64_t* abort_step) {
    if (!ctx || !prm || !mt || !rates || !states) return BC_ERR_INVALID_ARGUMENT;
    if (abort_step) *abort_step = -1;
    return guarded(ctx, [&]() -> int {
        // simulate.cpp:75-83
        if (prm->cells < 1) fail(BC_ERR_INVALID_ARGUMENT, "run_simulation: cells must be >= 1");
        if (!(prm->dt_seconds > 0.0)) fail(BC_ERR_INVALID_ARGUMENT, "run_simulation: dt must be positive");
        if (mt->species < 1 || mt->reactions < 0 || mt->nnz < 1 || mt->stamps < 0)
            fail(BC_ERR_INVALID_ARGUMENT, "run_simulation: bad mechanism tables");
        if (prm->steps > 0 && !per_step) fail(BC_ERR_INVALID_ARGUMENT, "run_simulation: per_step is NULL");
        const int64_t cells = prm->cells, s = mt->species, nnz = mt->nnz, R = mt->reactions;
        cudaStream_t st = static_cast<cudaStream_t>(prm->stream);

        // the pattern (kept when unchanged: plans and schedules survive)
        const bc::Pattern want = make_pattern(static_cast<int32_t>(s), mt->row_ptr, mt->col_idx);
        if (!ctx->has_pattern || ctx->pat.row_ptr != want.row_ptr || ctx->pat.col_idx != want.col_idx) {
            const int stp = bc_set_pattern(ctx, static_cast<int32_t>(s), mt->row_ptr, mt->col_idx);
            if (stp != BC_OK) throw Status(stp, ctx->err);
        }
        // evaluator tables -> device, one int32 buffer
        const int32_t nre = mt->reactant_ptr[R], npr = mt->product_ptr[R];
        std::vector<int32_t> tabs;
        auto put = [&](const int32_t* p, int64_t n) {
            const size_t at = tabs.size();
            tabs.insert(tabs.end(), p, p + n);
            return at;
        };
        const size_t o_sp = put(mt->stamp_ptr, R + 1), o_ss = put(mt->stamp_slot, mt->stamps),
                     o_so = put(mt->stamp_other, mt->stamps), o_rp = put(mt->reactant_ptr, R + 1),
                     o_re = put(mt->reactants, nre), o_pp = put(mt->product_ptr, R + 1),
                     o_pr = put(mt->products, npr), o_dg = put(mt->diag_slot, s);
        check_cuda(ctx->sim_tabs.ensure(sizeof(int32_t) * tabs.size()), "cudaMalloc");
        check_cuda(ctx->sim_sign.ensure(sizeof(double) * std::max<int64_t>(mt->stamps, 1)), "cudaMalloc");
        check_cuda(ctx->sim_rates.ensure(sizeof(double) * std::max<int64_t>(cells * R, 1)), "cudaMalloc");
        const size_t yb = sizeof(double) * cells * s;
        for (DevBuf* b : {&ctx->sim_y, &ctx->sim_prev, &ctx->sim_rhs, &ctx->sim_dx}) check_cuda(b->ensure(yb), "cudaMalloc");
        check_cuda(ctx->sim_values.ensure(sizeof(double) * cells * nnz), "cudaMalloc");
        check_cuda(ctx->sim_red.ensure(3 * sizeof(unsigned long long)), "cudaMalloc");
        check_cuda(ctx->f_scratch.ensure(yb), "cudaMalloc");
        check_cuda(cudaMemcpyAsync(ctx->sim_tabs.p, tabs.data(), sizeof(int32_t) * tabs.size(),
                                   cudaMemcpyHostToDevice, st), "H2D tables");
        if (mt->stamps > 0)
            check_cuda(cudaMemcpyAsync(ctx->sim_sign.p, mt->stamp_sign, sizeof(double) * mt->stamps,
                                       cudaMemcpyHostToDevice, st), "H2D signs");
        if (R > 0)
            check_cuda(cudaMemcpyAsync(ctx->sim_rates.p, rates, sizeof(double) * cells * R, cudaMemcpyDefault, st),
                       "H2D rates");
        double* y = ctx->sim_y.as<double>();
        double* yprev = ctx->sim_prev.as<double>();
        double* dx = ctx->sim_dx.as<double>();
        check_cuda(cudaMemcpyAsync(y, states, yb, cudaMemcpyDefault, st), "H2D states");
        const int32_t* tb = ctx->sim_tabs.as<int32_t>();
        const bc::NewtonParams np{cells, static_cast<int>(s), static_cast<int>(R), static_cast<int>(nnz),
                                  ctx->sim_rates.as<double>(), tb + o_sp, tb + o_ss, tb + o_so,
                                  ctx->sim_sign.as<double>(), tb + o_rp, tb + o_re, tb + o_pp, tb + o_pr, tb + o_dg,
                                  prm->dt_seconds, y, yprev, ctx->sim_values.as<double>(), ctx->sim_rhs.as<double>(),
                                  ctx->f_scratch.as<double>()};
        const unsigned asm_blocks = static_cast<unsigned>((cells + 127) / 128);
        const int64_t ny = cells * s;
        const unsigned ew_blocks = static_cast<unsigned>(std::min<int64_t>((ny + 255) / 256, 8 * ctx->sms));
        unsigned long long* red = ctx->sim_red.as<unsigned long long>();

        bc_solve_params sp{};
        sp.strategy = prm->strategy;
        sp.algo = prm->algo;
        sp.cells_per_block = prm->cells_per_block;
        sp.cells = cells;
        sp.tol = prm->tol;
        sp.max_iter = prm->max_iter;
        sp.max_threads_per_block = prm->max_threads_per_block;
        sp.stream = prm->stream;

        using Clock = std::chrono::steady_clock;
        for (int64_t step = 0; step < prm->steps; ++step) {  // simulate.cpp:103-176
            check_cuda(cudaMemcpyAsync(yprev, y, yb, cudaMemcpyDeviceToDevice, st), "D2D prev");
            bc_step_stats stats{};
            stats.step = step;
            for (int64_t newton = 1; newton <= prm->max_newton_iterations; ++newton) {
                bc::newton_assemble_kernel<<<asm_blocks, 128, 0, st>>>(np);
                check_cuda(cudaGetLastError(), "newton_assemble_kernel launch");
                ctx->launches++;
                if (prm->use_direct_reference) {  // lu_solve per cell (simulate.cpp:119-133)
                    const auto t0 = Clock::now();
                    std::vector<bc::LuEntry> ents(static_cast<size_t>(cells));
                    for (int64_t c = 0; c < cells; ++c) ents[c] = {c, c, 1, 0};
                    run_lu(ctx, ents, ctx->sim_values.as<double>(), ctx->sim_rhs.as<double>(), dx, nullptr,
                           static_cast<int>(s), static_cast<int>(nnz), 0, st);
                    stats.wall_time_ns +=
                        std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count();
                } else {  // run_strategy (simulate.cpp:134-147)
                    bc_report rep{};
                    const auto t0 = Clock::now();
                    const int rc = bc_solve(ctx, &sp, ctx->sim_values.as<double>(), ctx->sim_rhs.as<double>(), dx,
                                            nullptr, nullptr, nullptr, &rep);
                    const int64_t wall =
                        std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count();
                    if (rc != BC_OK) throw Status(rc, ctx->err);
                    stats.iterations_effective += rep.iterations_effective;
                    stats.iterations_sum += rep.iterations_sum;
                    stats.max_residual_rms = std::max(stats.max_residual_rms, rep.max_residual_rms);
                    stats.wall_time_ns += wall;
                    stats.breakdown_fallbacks += rep.breakdown_fallbacks;
                }
                // y += dy; |dy|_inf, |y|_inf, non-finite count (simulate.cpp:139-164)
                check_cuda(cudaMemsetAsync(red, 0, 3 * sizeof(unsigned long long), st), "memset");
                bc::newton_update_kernel<<<ew_blocks, 256, 0, st>>>(bc::UpdateParams{ny, y, dx, red});
                check_cuda(cudaGetLastError(), "newton_update_kernel launch");
                ctx->launches++;
                unsigned long long h[3];
                check_cuda(cudaMemcpyAsync(h, red, sizeof h, cudaMemcpyDeviceToHost, st), "D2H norms");
                check_cuda(cudaStreamSynchronize(st), "newton update");
                stats.newton_iterations = newton;
                if (h[2]) {
                    if (abort_step) *abort_step = step;
                    fail(BC_ERR_SOLVER_ABORT, "non-finite concentration at step " + std::to_string(step));
                }
                double update_inf, state_inf;
                std::memcpy(&update_inf, &h[0], 8);
                std::memcpy(&state_inf, &h[1], 8);
                if (update_inf < prm->newton_rtol * state_inf) break;
            }
            check_cuda(cudaMemsetAsync(red, 0, sizeof(unsigned long long), st), "memset");
            bc::clip_kernel<<<ew_blocks, 256, 0, st>>>(ny, y, red);
            check_cuda(cudaGetLastError(), "clip_kernel launch");
            ctx->launches++;
            unsigned long long clips = 0;
            check_cuda(cudaMemcpyAsync(&clips, red, sizeof clips, cudaMemcpyDeviceToHost, st), "D2H clips");
            check_cuda(cudaStreamSynchronize(st), "clip");
            stats.clip_events = static_cast<int64_t>(clips);
            per_step[step] = stats;
        }
        check_cuda(cudaMemcpyAsync(states, y, yb, cudaMemcpyDefault, st), "D2H states");
        check_cuda(cudaStreamSynchronize(st), "states");
        return BC_OK;
    });
}

}  // extern "C"
