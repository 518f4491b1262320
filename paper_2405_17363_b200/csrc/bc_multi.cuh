// bc_multi.cuh -- the Multi-cells strategy (K2, comparison baseline) and the
// general multi-interval ReductionPlan path of bicg_solve.
//
// One global block-diagonal system over cells*species unknowns
// (strategies.cpp:176-194), solved by ONE cooperative persistent kernel:
//   * the reduction plan's intervals (1024 rows each for Multi-cells,
//     exec_model.cpp:202-220; arbitrary for bicg_solve) are distributed over
//     the CTAs; a CTA computes every row-wise update of its intervals and the
//     interval's stride-halving tree in shared memory (reduction.cpp:38-44);
//   * grid.sync() separates phases whose SpMV reads rows owned by other CTAs;
//   * every CTA then folds all interval partials left to right -- the
//     reference's sequential host stage (reduction.hpp:68-77) -- so all CTAs
//     hold bit-identical scalars without a broadcast.
// This is the paper's Multi-cells arrangement: streaming
// vectors through HBM every iteration, grid-wide synchronisation, a
// sequential combine per reduction.  It is deliberately not fused like K1.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "bc_block.cuh"

namespace bc {

struct MultiParams {
    const double* values;   // cells * nnz
    const double* rhs;      // n
    const double* x0;       // n or nullptr
    double* x;              // n (solution, in/out)
    const int32_t* row_ptr; // pattern, species+1
    const int32_t* col_idx;
    const int32_t* trow_ptr;  // transpose pattern: per local column, entries in ascending row order
    const int32_t* trow;      //   source row
    const int32_t* tval;      //   value index
    const int32_t* diag;      // per species row: value index of the diagonal, -1 if none
    const int64_t* ranges;    // n_blocks * 2: reduction intervals
    int64_t n_blocks;
    int64_t n;
    int species, nnz;
    int max_len;              // longest interval (<= 4096)
    double* work;             // 9 * n doubles
    double* partials;         // n_blocks * 2
    double tol;
    int64_t max_iter;
    int algo;                 // 0 BiCG, 1 Jacobi-BiCGSTAB
    int mode;                 // 0 solve, 1 residual of x only
    int64_t* out_iters;
    double* out_rms;
    int32_t* out_flags;
    int stage_len;            // doubles per staging area (2 areas after the slots), 0 = none
};

namespace cgm = cooperative_groups;

struct MultiCtx {
    const MultiParams* p;
    double* slots;   // 2 * pow2(max_len) doubles (dynamic smem)
    double* red;     // small smem for broadcasts
    int P2;          // slots per value
    double* stage;   // 2 * stage_len doubles after the slots: gathered vectors of an interval's cells
};

// The gathered vectors were written by other CTAs before the last grid sync.
// An interval's rows only gather from their own cells (the system is block
// diagonal), so those cells' entries are staged into shared memory with
// coherent L2 reads (ld.global.cg, coalesced) and gathered from there; a
// plain L1-cached gather could return a line cached before the sync (under
// compute-sanitizer racecheck it did).  Returns the vector index of
// stage[0], or -1 when the cells do not fit (the row then reads through L2).
__device__ int64_t mc_stage(const MultiCtx& m, int area, const double* xin, int64_t r0, int64_t r1) {
    const MultiParams& p = *m.p;
    const int64_t c0 = r0 / p.species, c1 = (r1 - 1) / p.species;
    const int64_t base = c0 * p.species, cnt = (c1 - c0 + 1) * p.species;
    if (cnt > p.stage_len) return -1;
    double* st = m.stage + static_cast<int64_t>(area) * p.stage_len;
    __syncthreads();  // the previous interval's gathers are done
    for (int64_t q = threadIdx.x; q < cnt; q += blockDim.x) st[q] = __ldcg(xin + base + q);
    __syncthreads();
    return base;
}

// Row i of A x (csr.cpp:90-101) / of A^T x (csr.cpp:129-142): x from the
// staged copy (off >= 0, see mc_stage) or through L2.
__device__ __forceinline__ double mc_spmv_row(const MultiCtx& m, int area, int64_t off, int64_t i,
                                              const double* xin) {
    const MultiParams& p = *m.p;
    const int64_t c = i / p.species;
    const int r = static_cast<int>(i - c * p.species);
    const double* v = p.values + c * p.nnz;
    double acc = 0.0;
    if (off >= 0) {
        const double* xc = m.stage + static_cast<int64_t>(area) * p.stage_len + (c * p.species - off);
        for (int e = p.row_ptr[r]; e < p.row_ptr[r + 1]; ++e) acc = dadd(acc, dmul(v[e], xc[p.col_idx[e]]));
    } else {
        const double* xc = xin + c * p.species;
        for (int e = p.row_ptr[r]; e < p.row_ptr[r + 1]; ++e)
            acc = dadd(acc, dmul(v[e], __ldcg(xc + p.col_idx[e])));
    }
    return acc;
}

__device__ __forceinline__ double mc_spmvt_row(const MultiCtx& m, int area, int64_t off, int64_t j,
                                               const double* xin) {
    const MultiParams& p = *m.p;
    const int64_t c = j / p.species;
    const int lc = static_cast<int>(j - c * p.species);
    const double* v = p.values + c * p.nnz;
    double acc = 0.0;
    if (off >= 0) {
        const double* xc = m.stage + static_cast<int64_t>(area) * p.stage_len + (c * p.species - off);
        for (int q = p.trow_ptr[lc]; q < p.trow_ptr[lc + 1]; ++q) acc = dadd(acc, dmul(v[p.tval[q]], xc[p.trow[q]]));
    } else {
        const double* xc = xin + c * p.species;
        for (int q = p.trow_ptr[lc]; q < p.trow_ptr[lc + 1]; ++q)
            acc = dadd(acc, dmul(v[p.tval[q]], __ldcg(xc + p.trow[q])));
    }
    return acc;
}

// Partials of NV per-row values over this CTA's intervals: slot value of row
// i comes from f(i, v); tree in shared memory; partials[b*2+v].
template <int NV, class F>
__device__ void mc_block_partials(const MultiCtx& m, F&& f, const double* xin = nullptr) {
    const MultiParams& p = *m.p;
    for (int64_t b = blockIdx.x; b < p.n_blocks; b += gridDim.x) {
        const int64_t b0 = p.ranges[2 * b], len = p.ranges[2 * b + 1] - b0;
        const int64_t off = xin ? mc_stage(m, 0, xin, b0, b0 + len) : -1;  // f's SpMV gathers (fresh residual)
        int P = 1;
        while (P < len) P <<= 1;
        for (int q = threadIdx.x; q < P; q += blockDim.x)
#pragma unroll
            for (int v = 0; v < NV; ++v) m.slots[v * m.P2 + q] = q < len ? f(b0 + q, v, off) : 0.0;
        for (int stride = P / 2; stride >= 1; stride /= 2) {
            __syncthreads();
            for (int q = threadIdx.x; q < stride; q += blockDim.x)
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    m.slots[v * m.P2 + q] = dadd(m.slots[v * m.P2 + q], m.slots[v * m.P2 + q + stride]);
        }
        __syncthreads();
        if (threadIdx.x == 0)
#pragma unroll
            for (int v = 0; v < NV; ++v) p.partials[b * 2 + v] = m.slots[v * m.P2];
        __syncthreads();
    }
}

// The sequential left-to-right combine (reduction.hpp:68-77), done by every
// CTA so that all of them hold the same totals.  Partials are staged through
// shared memory in chunks; thread 0 folds them in order.
template <int NV>
__device__ void mc_combine(const MultiCtx& m, double (&tot)[NV]) {
    const MultiParams& p = *m.p;
    double acc[NV];
    const int chunk = m.P2;
    for (int64_t c0 = 0; c0 < p.n_blocks; c0 += chunk) {
        const int cnt = static_cast<int>(p.n_blocks - c0 < chunk ? p.n_blocks - c0 : chunk);
        __syncthreads();
        for (int q = threadIdx.x; q < cnt; q += blockDim.x)
#pragma unroll
            for (int v = 0; v < NV; ++v) m.slots[v * m.P2 + q] = __ldcg(p.partials + (c0 + q) * 2 + v);
        __syncthreads();
        if (threadIdx.x == 0)
            for (int q = 0; q < cnt; ++q)
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const double part = m.slots[v * m.P2 + q];
                    acc[v] = (c0 + q == 0) ? part : dadd(acc[v], part);
                }
    }
    if (threadIdx.x == 0)
#pragma unroll
        for (int v = 0; v < NV; ++v) m.red[v] = acc[v];
    __syncthreads();
#pragma unroll
    for (int v = 0; v < NV; ++v) tot[v] = m.red[v];
    __syncthreads();
}

// grid.sync() then a gpu-scope acquire fence: the next phase's plain loads of
// vectors other CTAs wrote must not hit a stale L1 line (compute-sanitizer
// racecheck's execution exposed exactly that without the fence).
__device__ __forceinline__ void mc_sync(cgm::grid_group& grid) {
    grid.sync();
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

template <class F>
__device__ __forceinline__ void mc_rows(const MultiParams& p, F&& f) {
    // rows of this CTA's intervals (so reductions never wait on other CTAs)
    for (int64_t b = blockIdx.x; b < p.n_blocks; b += gridDim.x)
        for (int64_t i = p.ranges[2 * b] + threadIdx.x; i < p.ranges[2 * b + 1]; i += blockDim.x) f(i);
}

// The same, with the interval's cells of x0 (and x1) staged first: f(i, off0, off1).
template <class F>
__device__ __forceinline__ void mc_rows_x(const MultiCtx& m, const double* x0, const double* x1, F&& f) {
    const MultiParams& p = *m.p;
    for (int64_t b = blockIdx.x; b < p.n_blocks; b += gridDim.x) {
        const int64_t r0 = p.ranges[2 * b], r1 = p.ranges[2 * b + 1];
        const int64_t off0 = mc_stage(m, 0, x0, r0, r1);
        const int64_t off1 = x1 ? mc_stage(m, 1, x1, r0, r1) : -1;
        for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) f(i, off0, off1);
    }
}

// fresh residual: sqrt(plan_reduce((b - A x)^2) / n)  (bicg.cpp:61-72)
__device__ double mc_fresh_rms(const MultiCtx& m, cgm::grid_group& grid) {
    const MultiParams& p = *m.p;
    mc_sync(grid);  // x complete
    mc_block_partials<1>(m, [&](int64_t i, int, int64_t off) {
        const double ri = dsub(p.rhs[i], mc_spmv_row(m, 0, off, i, p.x));
        return dmul(ri, ri);
    }, p.x);
    mc_sync(grid);
    double t[1];
    mc_combine<1>(m, t);
    return __dsqrt_rn(ddiv(t[0], static_cast<double>(p.n)));
}

__global__ void __launch_bounds__(256) multi_cells_kernel(const MultiParams p) {
    extern __shared__ __align__(16) double mc_smem[];
    __shared__ double s_red[4];
    cgm::grid_group grid = cgm::this_grid();
    MultiCtx m;
    m.p = &p;
    m.slots = mc_smem;
    m.red = s_red;
    m.P2 = 1;
    while (m.P2 < p.max_len) m.P2 <<= 1;
    if (m.P2 < 256) m.P2 = 256;
    m.stage = mc_smem + 2 * m.P2;
    const int64_t n = p.n;
    double* r = p.work;
    double* rh = r + n;   // BiCG: r~
    double* pv = rh + n;  // p
    double* v = pv + n;   // BiCGSTAB: v      BiCG: p~
    double* y = v + n;    // BiCGSTAB: y / z  BiCG: A p
    double* t = y + n;    // BiCGSTAB: t      BiCG: A^T p~
    double* dinv = t + n;
    const double nd = static_cast<double>(n);

    if (p.mode == 1) {  // residual of the given x only (LU fallback)
        const double f = mc_fresh_rms(m, grid);
        if (blockIdx.x == 0 && threadIdx.x == 0) *p.out_rms = f;
        return;
    }
    // setup (bicg.cpp:74-91): x = x0, r = 1*b + (-1)*A x
    mc_rows(p, [&](int64_t i) { p.x[i] = p.x0 ? p.x0[i] : 0.0; });
    mc_sync(grid);
    mc_rows_x(m, p.x, nullptr, [&](int64_t i, int64_t off, int64_t) {
        const double ri = dadd(p.rhs[i], -mc_spmv_row(m, 0, off, i, p.x));
        r[i] = ri;
        rh[i] = ri;
        if (p.algo == kBiCGStab) {
            pv[i] = 0.0;
            v[i] = 0.0;
            const int64_t c = i / p.species;
            const int lr = static_cast<int>(i - c * p.species);
            const int di = p.diag[lr];
            const double d = di >= 0 ? p.values[c * p.nnz + di] : 0.0;
            dinv[i] = d != 0.0 ? ddiv(1.0, d) : 1.0;
        } else {
            pv[i] = ri;
            v[i] = ri;
        }
    });
    // sigma = <r,r>, rho = <r~,r> from this CTA's rows only: no sync needed
    mc_block_partials<2>(m, [&](int64_t i, int w, int64_t) { return w == 0 ? dmul(r[i], r[i]) : dmul(rh[i], r[i]); });
    mc_sync(grid);
    double tot[2];
    mc_combine<2>(m, tot);
    double sigma = tot[0], rho_next = tot[1];
    int64_t iters = 0;
    bool conv = false, brk = false;
    double fres = 0.0;
    if (__dsqrt_rn(ddiv(sigma, nd)) <= p.tol) {
        fres = mc_fresh_rms(m, grid);
        conv = fres <= p.tol;
    }
    if (!conv) {
        double rho_prev = p.algo == kBiCGStab ? 1.0 : 0.0, alpha = 1.0, omega = 1.0;
        for (int64_t it = 1; it <= p.max_iter; ++it) {
            const double rho = rho_next;
            if (scalar_breaks(rho)) { brk = true; break; }
            if (p.algo == kBiCGStab) {
                const double beta = dmul(ddiv(rho, rho_prev), ddiv(alpha, omega));
                mc_rows(p, [&](int64_t i) {
                    pv[i] = dadd(r[i], dmul(beta, dsub(pv[i], dmul(omega, v[i]))));
                    y[i] = dmul(dinv[i], pv[i]);
                });
                mc_sync(grid);
                mc_rows_x(m, y, nullptr, [&](int64_t i, int64_t off, int64_t) { v[i] = mc_spmv_row(m, 0, off, i, y); });
                mc_block_partials<1>(m, [&](int64_t i, int, int64_t) { return dmul(rh[i], v[i]); });
                mc_sync(grid);
                double d1[1];
                mc_combine<1>(m, d1);
                if (scalar_breaks(d1[0])) { brk = true; break; }
                alpha = ddiv(rho, d1[0]);
                mc_rows(p, [&](int64_t i) {
                    r[i] = dsub(r[i], dmul(alpha, v[i]));  // r <- s
                    p.x[i] = dadd(p.x[i], dmul(alpha, y[i]));
                    y[i] = dmul(dinv[i], r[i]);           // y <- z
                });
                mc_sync(grid);
                mc_rows_x(m, y, nullptr, [&](int64_t i, int64_t off, int64_t) { t[i] = mc_spmv_row(m, 0, off, i, y); });
                mc_block_partials<2>(m, [&](int64_t i, int w, int64_t) { return w == 0 ? dmul(t[i], t[i]) : dmul(t[i], r[i]); });
                mc_sync(grid);
                double d2[2];
                mc_combine<2>(m, d2);
                const double tt = d2[0], ts = d2[1];
                if (tt != 0.0 && scalar_breaks(tt)) { brk = true; break; }
                omega = tt == 0.0 ? 0.0 : ddiv(ts, tt);
                mc_rows(p, [&](int64_t i) {
                    p.x[i] = dadd(p.x[i], dmul(omega, y[i]));
                    r[i] = dsub(r[i], dmul(omega, t[i]));
                });
            } else {
                if (it > 1) {
                    const double beta = ddiv(rho, rho_prev);
                    mc_rows(p, [&](int64_t i) {
                        pv[i] = dadd(r[i], dmul(beta, pv[i]));
                        v[i] = dadd(rh[i], dmul(beta, v[i]));
                    });
                }
                mc_sync(grid);
                mc_rows_x(m, pv, v, [&](int64_t i, int64_t off0, int64_t off1) {
                    y[i] = mc_spmv_row(m, 0, off0, i, pv);
                    t[i] = mc_spmvt_row(m, 1, off1, i, v);
                });
                mc_block_partials<1>(m, [&](int64_t i, int, int64_t) { return dmul(v[i], y[i]); });
                mc_sync(grid);
                double d1[1];
                mc_combine<1>(m, d1);
                if (scalar_breaks(d1[0])) { brk = true; break; }
                alpha = ddiv(rho, d1[0]);
                const double nalpha = -alpha;
                mc_rows(p, [&](int64_t i) {
                    p.x[i] = dadd(p.x[i], dmul(alpha, pv[i]));
                    r[i] = dadd(r[i], dmul(nalpha, y[i]));
                    rh[i] = dadd(rh[i], dmul(nalpha, t[i]));
                });
            }
            rho_prev = rho;
            iters = it;
            mc_block_partials<2>(m, [&](int64_t i, int w, int64_t) { return w == 0 ? dmul(r[i], r[i]) : dmul(rh[i], r[i]); });
            mc_sync(grid);
            mc_combine<2>(m, tot);
            sigma = tot[0];
            rho_next = tot[1];
            if (!isfinite(sigma)) { brk = true; break; }
            if (__dsqrt_rn(ddiv(sigma, nd)) <= p.tol) {
                const double f = mc_fresh_rms(m, grid);
                if (f <= p.tol) {
                    fres = f;
                    conv = true;
                    break;
                }
            }
            if (p.algo == kBiCGStab && scalar_breaks(omega)) { brk = true; break; }
        }
        if (!conv) {
            fres = mc_fresh_rms(m, grid);
            conv = !brk && fres <= p.tol;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *p.out_iters = iters;
        *p.out_rms = fres;
        *p.out_flags = (conv ? 1 : 0) | (brk ? 2 : 0);
    }
}

}  // namespace bc
