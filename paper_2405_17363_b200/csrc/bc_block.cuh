// bc_block.cuh -- the fused, persistent Block-cells solve kernel (K1).
//
// One team of W warps owns one group of k cells (k*species rows) at a time
// and runs the whole Krylov solve for it on-chip: values staged once into
// shared memory in SpMV-schedule order, working vectors in registers (each
// lane owns RV row slots), the gather vector and SpMV outputs in shared
// memory, reductions with a per-lane tree + (W>1) one cross-warp shared
// step + an xor butterfly, and the convergence test inside the team.  There
// is no grid-wide synchronisation and no host round trip per iteration.
// Teams fetch groups from an atomic counter (dynamic load balance for the
// converging regime).
//
// Floating point follows the reference bit for bit: every
// product/sum is an explicit __dmul_rn/__dadd_rn/__dsub_rn (no FMA
// contraction), SpMV rows accumulate from 0.0 in CSR order (csr.cpp:90-101),
// A^T products accumulate in ascending row order (csr.cpp:129-142), and
// reductions reproduce tree_reduce_in_place (reduction.cpp:38-44).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bc_plan.hpp"

namespace bc {

enum AlgoKind { kBiCG = 0, kBiCGStab = 1 };

// Host inputs streamed in while the kernel runs (bc_solve): the copy engine
// writes chunk c's values and rhs, then ready[c] = 1.  Group g of a launch
// belongs to chunk chunk_base + g / chunk_groups; chunk boundaries fall on
// 128-byte lines, so no line of a chunk is cached before its flag is seen.
struct InputGate {
    const unsigned int* ready;
    unsigned int* err;  // set if a chunk never arrives (a stalled copy engine)
    int chunk_groups, chunk_base;
};

struct BlockParams {
    const double* values;   // cells * nnz
    const double* rhs;      // cells * species
    const double* x0;       // cells * species or nullptr (zeros)
    double* x_out;          // cells * species
    int32_t* g_iters;
    double* g_rms;
    uint8_t* g_flags;
    const uint32_t* words;  // A schedule, S * LW
    const uint32_t* twords; // A^T schedule, St * LW (BiCG)
    const int32_t* vpos;    // k*nnz
    const int32_t* tvpos;   // k*nnz (BiCG)
    const int32_t* dpos;    // n (BiCGSTAB)
    unsigned int* counter;  // work counter (zeroed before launch)
    int64_t cell_offset;    // first cell of group 0 of this launch
    int64_t group_offset;   // output index of group 0 of this launch
    int group_count;
    int n, species, nnz, kc;
    int S, St, P;
    int teams;              // teams per CTA
    int team_doubles;       // shared doubles per team
    int sched_words;        // shared u32 words of schedules per CTA (padded to even)
    double tol;
    int64_t max_iter;
    // Staging level for groups too large for shared memory (comparison
    // strategies only; Block-cells(1) at CB05 size is always level 0):
    //   0: schedules and values in shared memory
    //   1: schedules read from global (L1/L2-resident), values in shared memory
    //   2: schedules and values read from global, values through vidx/tvidx
    int level;
    const int32_t* vidx;    // schedule slot -> group value index (level 2)
    const int32_t* tvidx;
    const int32_t* didx;    // group row -> group value index of the diagonal, -1 if none
    const int32_t* xpos;    // group row -> shared slot of the gathered vector (A pass)
    const int32_t* txpos;   // same for the A^T pass (BiCG)
    int xslots, txslots;    // shared slots of the gathered vectors (multiples of 32)
    InputGate gate;         // streamed host inputs (bc_solve), or gate.ready == nullptr
};

// One thread waits for group g's chunk (acquire), the caller then syncs its team.
__device__ __forceinline__ void gate_wait(const InputGate& gt, int g) {
    if (!gt.ready) return;
    const unsigned int* f = gt.ready + gt.chunk_base + g / gt.chunk_groups;
    const long long t0 = clock64();
    for (;;) {
        unsigned int v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v) break;
        if (clock64() - t0 > (20ll << 30)) {  // ~10 s at 2 GHz
            atomicExch(gt.err, 1u);
            break;
        }
        __nanosleep(500);
    }
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// bicg.cpp:12-14
__device__ __forceinline__ bool scalar_breaks(double v) { return !isfinite(v) || fabs(v) < 1e-300; }

template <int W>
struct Team {
    int w, lane, tid, id;
    __device__ __forceinline__ void sync() const {
        if constexpr (W == 1) {
            __syncwarp();
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(W * 32) : "memory");
        }
    }
};

template <int W, int R, int RV>
struct Ctx {
    Team<W> tm;
    int n, P;
    double* Xs;   // gather source, row(j) stored at slot xa[j]
    double* Xs2;  // second gather source (BiCG: p~), row(j) at slot xt[j]
    int xa[RV], xt[RV];
    double* Ys;   // A products
    double* Yt;   // A^T products (BiCG)
    double* red;  // cross-warp partials [2][4][W][32]
    int red_buf;
    // SpMV operands: schedule words, values (schedule order, or indexed), steps
    const uint32_t* Wa;
    const double* Va;
    const int32_t* Ia;
    int Sa;
    const uint32_t* Wt;
    const double* Vt;
    const int32_t* It;
    int St;
    __device__ __forceinline__ int row(int j) const { return (j * W + tm.w) * 32 + tm.lane; }
    __device__ __forceinline__ bool valid(int j) const { return row(j) < n; }
};

// Reduce NV values over the group.  vals[v][j] is the slot
// value of row(j); invalid rows contribute an explicit +0.0 exactly as the
// reference's zero-padded slots do.
template <int NV, int W, int R, int RV>
__device__ __forceinline__ void team_reduce(Ctx<W, R, RV>& c, const double (&vals)[NV][RV],
                                            double (&out)[NV]) {
    double part[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        double t[R];
#pragma unroll
        for (int j = 0; j < R; ++j) t[j] = (j < RV && c.valid(j)) ? vals[v][j < RV ? j : 0] : 0.0;
#pragma unroll
        for (int stride = R / 2; stride >= 1; stride /= 2)
#pragma unroll
            for (int j = 0; j < stride; ++j) t[j] = dadd(t[j], t[j + stride]);
        part[v] = t[0];
    }
    if constexpr (W > 1) {
        double* buf = c.red + c.red_buf * (4 * W * 32);
#pragma unroll
        for (int v = 0; v < NV; ++v) buf[(v * W + c.tm.w) * 32 + c.tm.lane] = part[v];
        c.tm.sync();
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double u[W];
#pragma unroll
            for (int q = 0; q < W; ++q) u[q] = buf[(v * W + q) * 32 + c.tm.lane];
#pragma unroll
            for (int stride = W / 2; stride >= 1; stride /= 2)
#pragma unroll
                for (int q = 0; q < stride; ++q) u[q] = dadd(u[q], u[q + stride]);
            part[v] = u[0];
        }
        c.red_buf ^= 1;
    }
    if (c.P >= 32) {
#pragma unroll
        for (int mask = 16; mask >= 1; mask >>= 1)
#pragma unroll
            for (int v = 0; v < NV; ++v) part[v] = dadd(part[v], __shfl_xor_sync(0xffffffffu, part[v], mask));
    } else {
        for (int mask = c.P / 2; mask >= 1; mask >>= 1)
#pragma unroll
            for (int v = 0; v < NV; ++v) part[v] = dadd(part[v], __shfl_xor_sync(0xffffffffu, part[v], mask));
#pragma unroll
        for (int v = 0; v < NV; ++v) part[v] = __shfl_sync(0xffffffffu, part[v], 0);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) out[v] = part[v];
}

// One schedule pass: every lane walks its segments, writing each finished
// row (column, for A^T) sum into Y.
template <int W, bool INDEXED>
__device__ __forceinline__ void sched_pass_impl(const uint32_t* __restrict__ words, const double* __restrict__ V,
                                                const int32_t* __restrict__ vidx, int steps, int L,
                                                const double* X, double* Y) {
    constexpr int LW = W * 32;
    double acc = 0.0;
#pragma unroll 4
    for (int t = 0; t < steps; ++t) {
        const uint32_t e = words[t * LW + L];
        const double a = INDEXED ? V[vidx[t * LW + L]] : V[t * LW + L];
        const double xv = X[e & kColMask];
        acc = dadd(acc, dmul(a, xv));
        if (e & kEndBit) {
            Y[(e >> kColBits) & kColMask] = acc;
            acc = 0.0;
        }
    }
}

template <int W>
__device__ __forceinline__ void sched_pass(const uint32_t* words, const double* V, const int32_t* vidx,
                                           int steps, int L, const double* X, double* Y) {
    if (vidx)
        sched_pass_impl<W, true>(words, V, vidx, steps, L, X, Y);
    else
        sched_pass_impl<W, false>(words, V, nullptr, steps, L, X, Y);
}

// y = A x over the group (csr.cpp:90-101 semantics).
template <int W, int R, int RV>
__device__ __forceinline__ void team_spmv(Ctx<W, R, RV>& c, const double (&x)[RV], double (&y)[RV]) {
#pragma unroll
    for (int j = 0; j < RV; ++j)
        if (c.valid(j)) c.Xs[c.xa[j]] = x[j];
    c.tm.sync();
    sched_pass<W>(c.Wa, c.Va, c.Ia, c.Sa, c.tm.tid, c.Xs, c.Ys);
    c.tm.sync();
#pragma unroll
    for (int j = 0; j < RV; ++j) y[j] = c.valid(j) ? c.Ys[c.row(j)] : 0.0;
}

// ap = A p and atps = A^T ps in one pass (BiCG, bicg.cpp:106-107).
template <int W, int R, int RV>
__device__ __forceinline__ void team_spmv_pair(Ctx<W, R, RV>& c, const double (&p)[RV], const double (&ps)[RV],
                                               double (&ap)[RV], double (&atps)[RV]) {
#pragma unroll
    for (int j = 0; j < RV; ++j)
        if (c.valid(j)) {
            c.Xs[c.xa[j]] = p[j];
            c.Xs2[c.xt[j]] = ps[j];
        }
    c.tm.sync();
    sched_pass<W>(c.Wa, c.Va, c.Ia, c.Sa, c.tm.tid, c.Xs, c.Ys);
    sched_pass<W>(c.Wt, c.Vt, c.It, c.St, c.tm.tid, c.Xs2, c.Yt);
    c.tm.sync();
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        ap[j] = c.valid(j) ? c.Ys[c.row(j)] : 0.0;
        atps[j] = c.valid(j) ? c.Yt[c.row(j)] : 0.0;
    }
}

// bicg.cpp:61-72 residual_rms: sqrt(tree((b - A x)^2) / n)
template <int W, int R, int RV>
__device__ __forceinline__ double fresh_rms(Ctx<W, R, RV>& c, const double (&x)[RV], const double (&b)[RV]) {
    double ax[RV];
    team_spmv(c, x, ax);
    double sq[1][RV];
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        const double ri = dsub(b[j], ax[j]);
        sq[0][j] = dmul(ri, ri);
    }
    double out[1];
    team_reduce<1>(c, sq, out);
    return __dsqrt_rn(ddiv(out[0], static_cast<double>(c.n)));
}

template <int ALGO, int W, int R, int RV>
__global__ void __launch_bounds__(256, 1) block_cells_kernel(const BlockParams p) {
    constexpr int LW = W * 32;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* s_words = reinterpret_cast<uint32_t*>(smem);
    uint32_t* s_twords = s_words + p.S * LW;
    double* team_base = reinterpret_cast<double*>(smem + sizeof(uint32_t) * p.sched_words);
    const bool words_smem = p.level == 0, values_smem = p.level < 2;

    // CTA-shared schedules (identical for every group)
    if (words_smem) {
        for (int i = threadIdx.x; i < p.S * LW; i += blockDim.x) s_words[i] = p.words[i];
        if constexpr (ALGO == kBiCG)
            for (int i = threadIdx.x; i < p.St * LW; i += blockDim.x) s_twords[i] = p.twords[i];
    }
    __syncthreads();

    const int team_id = threadIdx.x / LW;
    Ctx<W, R, RV> c;
    c.tm.id = team_id;
    c.tm.tid = threadIdx.x % LW;
    c.tm.w = c.tm.tid / 32;
    c.tm.lane = c.tm.tid % 32;
    c.n = p.n;
    c.P = p.P;
    const int n_pad = (p.n + 31) & ~31;
    double* Vs = team_base + static_cast<size_t>(team_id) * p.team_doubles;
    double* Vt = Vs + p.S * LW;
    double* tail = values_smem ? Vt + (ALGO == kBiCG ? p.St * LW : 0) : Vs;
    c.Xs = tail;
    c.Ys = tail + p.xslots;
    c.Xs2 = c.Ys + n_pad;
    c.Yt = c.Xs2 + (ALGO == kBiCG ? p.txslots : 0);
    c.red = c.Yt + (ALGO == kBiCG ? n_pad : 0);
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        c.xa[j] = c.valid(j) ? p.xpos[c.row(j)] : 0;
        c.xt[j] = (ALGO == kBiCG && c.valid(j)) ? p.txpos[c.row(j)] : 0;
    }
    c.red_buf = 0;
    c.Wa = words_smem ? s_words : p.words;
    c.Wt = words_smem ? s_twords : p.twords;
    c.Sa = p.S;
    c.St = p.St;
    c.Ia = values_smem ? nullptr : p.vidx;
    c.It = values_smem ? nullptr : p.tvidx;
    __shared__ int s_group[32];

    for (;;) {
        int gl;
        if constexpr (W == 1) {
            unsigned int v = 0;
            if (c.tm.lane == 0) v = atomicAdd(p.counter, 1u);
            gl = static_cast<int>(__shfl_sync(0xffffffffu, v, 0));
        } else {
            if (c.tm.tid == 0) s_group[team_id] = static_cast<int>(atomicAdd(p.counter, 1u));
            c.tm.sync();
            gl = s_group[team_id];
            c.tm.sync();
        }
        if (gl >= p.group_count) break;
        if (p.gate.ready) {
            if (c.tm.tid == 0) gate_wait(p.gate, gl);
            c.tm.sync();
        }

        const int64_t cell0 = p.cell_offset + static_cast<int64_t>(gl) * p.kc;
        const double* src = p.values + cell0 * p.nnz;
        const int cnt = p.kc * p.nnz;
        if (values_smem) {
            // stage this group's values into schedule order (once per solve)
            for (int e = c.tm.tid; e < cnt; e += LW) {
                const double a = __ldcs(src + e);
                Vs[p.vpos[e]] = a;
                if constexpr (ALGO == kBiCG) Vt[p.tvpos[e]] = a;
            }
            c.Va = Vs;
            c.Vt = Vt;
        } else {
            c.Va = src;  // level 2: read through vidx/tvidx (L1/L2)
            c.Vt = src;
        }
        for (int i = c.tm.tid; i < p.n; i += LW) {
            c.Ys[i] = 0.0;  // empty rows read +0.0, as spmv's sum = 0.0
            if constexpr (ALGO == kBiCG) c.Yt[i] = 0.0;
        }
        const double* bsrc = p.rhs + cell0 * p.species;
        double b[RV], x[RV];
#pragma unroll
        for (int j = 0; j < RV; ++j) {
            const bool ok = c.valid(j);
            b[j] = ok ? __ldcs(bsrc + c.row(j)) : 0.0;
            x[j] = (ok && p.x0) ? p.x0[cell0 * p.species + c.row(j)] : 0.0;
        }
        c.tm.sync();

        int64_t iters = 0;
        bool conv = false, brk = false;
        double fres = 0.0;
        const double nd = static_cast<double>(p.n);

        if constexpr (ALGO == kBiCGStab) {
            double dinv[RV];
#pragma unroll
            for (int j = 0; j < RV; ++j) {
                double d = 0.0;
                if (c.valid(j)) {
                    if (values_smem) {
                        const int dp = p.dpos[c.row(j)];
                        d = dp >= 0 ? Vs[dp] : 0.0;
                    } else {
                        const int di = p.didx[c.row(j)];
                        d = di >= 0 ? src[di] : 0.0;
                    }
                    dinv[j] = d != 0.0 ? ddiv(1.0, d) : 1.0;
                } else {
                    dinv[j] = 0.0;
                }
            }
            double r[RV], rh[RV], pv[RV], v[RV];
            {
                double ax[RV];
                team_spmv(c, x, ax);
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    r[j] = c.valid(j) ? dadd(b[j], -ax[j]) : 0.0;  // 1*b + (-1)*Ax
                    rh[j] = r[j];
                    pv[j] = 0.0;
                    v[j] = 0.0;
                }
            }
            double red2[2];
            {
                double q[2][RV];
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    q[0][j] = dmul(r[j], r[j]);
                    q[1][j] = dmul(rh[j], r[j]);
                }
                team_reduce<2>(c, q, red2);
            }
            if (__dsqrt_rn(ddiv(red2[0], nd)) <= p.tol) {
                fres = fresh_rms(c, x, b);
                conv = fres <= p.tol;
            }
            if (!conv) {
                double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
                double rho_next = red2[1];
                for (int64_t it = 1; it <= p.max_iter; ++it) {
                    const double rho = rho_next;
                    if (scalar_breaks(rho)) { brk = true; break; }
                    const double beta = dmul(ddiv(rho, rho_prev), ddiv(alpha, omega));
                    double y[RV];
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        pv[j] = dadd(r[j], dmul(beta, dsub(pv[j], dmul(omega, v[j]))));
                        y[j] = dmul(dinv[j], pv[j]);
                    }
                    team_spmv(c, y, v);
                    double den;
                    {
                        double q[1][RV], o[1];
#pragma unroll
                        for (int j = 0; j < RV; ++j) q[0][j] = dmul(rh[j], v[j]);
                        team_reduce<1>(c, q, o);
                        den = o[0];
                    }
                    if (scalar_breaks(den)) { brk = true; break; }
                    alpha = ddiv(rho, den);
                    double s[RV], z[RV];
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        s[j] = dsub(r[j], dmul(alpha, v[j]));
                        z[j] = dmul(dinv[j], s[j]);
                        x[j] = dadd(x[j], dmul(alpha, y[j]));
                    }
                    double t[RV];
                    team_spmv(c, z, t);
                    double tt, ts;
                    {
                        double q[2][RV], o[2];
#pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(t[j], t[j]);
                            q[1][j] = dmul(t[j], s[j]);
                        }
                        team_reduce<2>(c, q, o);
                        tt = o[0];
                        ts = o[1];
                    }
                    if (tt != 0.0 && scalar_breaks(tt)) { brk = true; break; }
                    omega = tt == 0.0 ? 0.0 : ddiv(ts, tt);
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        x[j] = dadd(x[j], dmul(omega, z[j]));
                        r[j] = dsub(s[j], dmul(omega, t[j]));
                    }
                    rho_prev = rho;
                    iters = it;
                    double sigma;
                    {
                        double q[2][RV], o[2];
#pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(r[j], r[j]);
                            q[1][j] = dmul(rh[j], r[j]);
                        }
                        team_reduce<2>(c, q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (__dsqrt_rn(ddiv(sigma, nd)) <= p.tol) {
                        const double f = fresh_rms(c, x, b);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                    if (scalar_breaks(omega)) { brk = true; break; }
                }
                if (!conv) {
                    fres = fresh_rms(c, x, b);
                    conv = !brk && fres <= p.tol;
                }
            }
        } else {
            // bicg.cpp:42-142
            double r[RV], rs[RV], pv[RV], ps[RV];
            {
                double ax[RV];
                team_spmv(c, x, ax);
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    r[j] = c.valid(j) ? dadd(b[j], -ax[j]) : 0.0;
                    rs[j] = r[j];
                    pv[j] = r[j];
                    ps[j] = r[j];
                }
            }
            double red2[2];
            {
                double q[2][RV];
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    q[0][j] = dmul(r[j], r[j]);
                    q[1][j] = dmul(rs[j], r[j]);
                }
                team_reduce<2>(c, q, red2);
            }
            if (__dsqrt_rn(ddiv(red2[0], nd)) <= p.tol) {
                fres = fresh_rms(c, x, b);
                conv = fres <= p.tol;
            }
            if (!conv) {
                double rho_prev = 0.0;
                double rho_next = red2[1];
                for (int64_t it = 1; it <= p.max_iter; ++it) {
                    const double rho = rho_next;
                    if (scalar_breaks(rho)) { brk = true; break; }
                    if (it > 1) {
                        const double beta = ddiv(rho, rho_prev);
#pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            pv[j] = dadd(r[j], dmul(beta, pv[j]));
                            ps[j] = dadd(rs[j], dmul(beta, ps[j]));
                        }
                    }
                    double ap[RV], atps[RV];
                    team_spmv_pair(c, pv, ps, ap, atps);
                    double den;
                    {
                        double q[1][RV], o[1];
#pragma unroll
                        for (int j = 0; j < RV; ++j) q[0][j] = dmul(ps[j], ap[j]);
                        team_reduce<1>(c, q, o);
                        den = o[0];
                    }
                    if (scalar_breaks(den)) { brk = true; break; }
                    const double alpha = ddiv(rho, den);
                    const double nalpha = -alpha;
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        x[j] = dadd(x[j], dmul(alpha, pv[j]));
                        r[j] = dadd(r[j], dmul(nalpha, ap[j]));
                        rs[j] = dadd(rs[j], dmul(nalpha, atps[j]));
                    }
                    rho_prev = rho;
                    iters = it;
                    double sigma;
                    {
                        double q[2][RV], o[2];
#pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(r[j], r[j]);
                            q[1][j] = dmul(rs[j], r[j]);
                        }
                        team_reduce<2>(c, q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (__dsqrt_rn(ddiv(sigma, nd)) <= p.tol) {
                        const double f = fresh_rms(c, x, b);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                }
                if (!conv) {
                    fres = fresh_rms(c, x, b);
                    conv = !brk && fres <= p.tol;
                }
            }
        }

        double* xdst = p.x_out + cell0 * p.species;
#pragma unroll
        for (int j = 0; j < RV; ++j)
            if (c.valid(j)) xdst[c.row(j)] = x[j];
        if (c.tm.tid == 0) {
            const int64_t g = p.group_offset + gl;
            p.g_iters[g] = static_cast<int32_t>(iters);
            p.g_rms[g] = fres;
            p.g_flags[g] = static_cast<uint8_t>((conv ? 1 : 0) | (brk ? 2 : 0));
        }
        c.tm.sync();
    }
}

}  // namespace bc
