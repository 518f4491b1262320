// bc_latency.cuh -- latency mode for small batches (BASELINE configs[0]: 100
// cells; batches that leave SMs idle): one CTA of RV = ceil(n/32) warps per
// group.
//
// The throughput kernel (bc_tmem.cuh) runs a cell on one warp (52 schedule
// steps per SpMV) and overlaps 16 cells per SM to fill the shared-memory
// pipe; alone on an SM one cell takes ~4.5 ms for 1000 iterations (~8,900
// cycles per iteration, a dependent-latency chain).  When there are fewer
// groups than SMs can overlap, latency is the metric.  Here warp 0 (the
// leader) holds the group's Krylov vectors in the throughput kernel's owner
// layout (lane l, slot j: row 32j + l -- so every dot product is
// tmem_reduce's lane tree + xor butterfly, the reference's stride-halving
// tree, in registers with no cross-warp step) and runs the scalar
// recurrences; the SpMV is split over all warps, one row per thread (the
// reference's own Block-cells geometry, exec_model.cpp:115-122, 134-158):
//
//   * the leader publishes the vector into the one shared gather region
//     (lane-major, conflict-free), posts the order (SpMV, SpMV pair, exit)
//     and arrives at barrier A;
//   * thread t computes the row the schedule gave it (rows dealt longest
//     first, so later warps run fewer steps; bc_latency_plan.cpp): its
//     values and gather offsets live in registers, entries in CSR order,
//     padding entries are (0.0, a zero slot) which add exact +0.0 to a sum
//     that started at +0.0 (csr.cpp:90-101 bit for bit);
//   * the row sums meet in Y at barrier B and the leader reads the product
//     back into its owner slots; the helper warps wait at the next A.
// Per Jacobi-BiCGSTAB iteration that is 4 block barriers; nothing but the
// row chains runs outside warp 0.  BiCG's A^T row runs beside the A row as a
// second chain over p~ (published at P + 16).  Rows >= n carry exact +0.0
// (dinv 0, values 0), as in bc_tmem.cuh.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bc_block.cuh"
#include "bc_tmem.cuh"  // lds64, tmem_reduce

namespace bc {

#ifdef BC_LAT_PROFILE
// phase timing (thread 0 of CTA 0): cumulative cycles per phase of an iteration
__device__ unsigned long long bc_lat_prof[16];
#define LAT_MARK(i)                      \
    do {                                 \
        const long long now = clock64(); \
        prof_acc[i] += now - prof_t;     \
        prof_t = now;                    \
    } while (0)
#else
#define LAT_MARK(i) \
    do {            \
    } while (0)
#endif

struct LatencyParams {
    const double* values;  // cells * nnz
    const double* rhs;     // cells * species
    double* x_out;
    int32_t* g_iters;
    double* g_rms;
    uint8_t* g_flags;
    // the schedule (bc_latency_plan.cpp), [L][T] tables indexed e * T + t
    const int32_t* rowof;  // [T] group row thread t computes in the SpMV, -1 none
    const int32_t* steps;  // [T] SpMV steps of thread t's warp
    const int32_t* rvi;    // group value index of the row's e-th entry, -1 = padding
    const uint16_t* rxo;   // byte offset of its gather slot in the warp's copy (padding: a zero slot)
    const int32_t* tvi;    // BiCG: the A^T row's entries (ascending source row)
    const uint16_t* txo;   // BiCG: byte offsets into the warp's p~ copy
    const int32_t* didx;   // [P] group value index of row i's diagonal, -1 if none / i >= n
    int64_t cell_offset, group_offset;
    int group_count;
    int n, nnz, P, species, kc;
    int xs;                // doubles of one warp's gather region (x | 16 zero slots | [p~])
    double sigma_max;      // sqrt(sigma/n) <= tol  <=>  sigma <= sigma_max
    double tol;
    int max_iter;
    InputGate gate;
};

template <int LMAX>
struct LatRow {
    double a[LMAX];
    uint32_t o[LMAX];
};

// y = sum_e a[e] * X[o[e]] in CSR order from +0.0 (gathers issued first),
// over NS steps (entries NS.. of the row are padding here).
template <int NS, int LMAX>
__device__ __forceinline__ double lat_row_n(const LatRow<LMAX>& rw, uint32_t xbase) {
    double g[NS];
#pragma unroll
    for (int e = 0; e < NS; ++e) g[e] = lds64(xbase + rw.o[e]);
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < NS; ++e) acc = dadd(acc, dmul(rw.a[e], g[e]));
    return acc;
}

// The warp's own step count: a warp-uniform choice among straight-line instances.
template <int LMAX>
__device__ __forceinline__ double lat_row(const LatRow<LMAX>& rw, uint32_t xbase, int nsteps) {
    if (nsteps <= 8) return lat_row_n<8, LMAX>(rw, xbase);
    if (nsteps <= 12) return lat_row_n<12, LMAX>(rw, xbase);
    if constexpr (LMAX > 16) {
        if (nsteps <= 16) return lat_row_n<16, LMAX>(rw, xbase);
        if (nsteps <= 20) return lat_row_n<20, LMAX>(rw, xbase);
    }
    if constexpr (LMAX > 24) {
        if (nsteps <= 24) return lat_row_n<24, LMAX>(rw, xbase);
        if (nsteps <= 28) return lat_row_n<28, LMAX>(rw, xbase);
    }
    return lat_row_n<LMAX, LMAX>(rw, xbase);
}

// Per-thread state of the split SpMV.
template <int RV, int LMAX>
struct LatWarp {
    double* X;        // the gather region (generic): x | 16 zero slots | [p~]
    uint32_t xaddr;   // its shared address
    double* Y;        // [2][P]: (A, A^T) row sums
    int P, lane, T;
    int srow;         // the row this thread computes, -1 none
    int nsteps;
    volatile int* ctrl;  // the leader's order to the helper warps: kLatSpmv / kLatPair / kLatExit
    LatRow<LMAX> ra;
};

constexpr int kLatSpmv = 1, kLatPair = 2, kLatExit = 3;

// The two block barriers of an SpMV: A (operands published, order posted)
// and B (row sums in Y).  Named, so that the leader and the helpers can reach
// them from different code.
__device__ __forceinline__ void lat_bar_a(int T) { asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory"); }
__device__ __forceinline__ void lat_bar_b(int T) { asm volatile("bar.sync 2, %0;" ::"r"(T) : "memory"); }

// y = A v, called by the leader (warp 0, which holds the Krylov vectors):
// publish v (owner slots, lane-major, conflict-free), post the order, every
// warp computes its rows (helpers in lat_helper), the leader reads the
// products back after the second barrier.
template <int RV, int LMAX>
__device__ __forceinline__ void lat_spmv(LatWarp<RV, LMAX>& lw, const double (&v)[RV], double (&y)[RV]) {
#pragma unroll
    for (int j = 0; j < RV; ++j) lw.X[j * 32 + lw.lane] = v[j];
    if (lw.lane == 0) *lw.ctrl = kLatSpmv;
    lat_bar_a(lw.T);
    const double s = lat_row<LMAX>(lw.ra, lw.xaddr, lw.nsteps);
    if (lw.srow >= 0) lw.Y[lw.srow] = s;
    lat_bar_b(lw.T);
#pragma unroll
    for (int j = 0; j < RV; ++j) y[j] = lw.Y[j * 32 + lw.lane];
}

// BiCG: A p and A^T p~ in one exchange (p~ published at offset P + 16).
template <int RV, int LMAX>
__device__ __forceinline__ void lat_spmv_pair(LatWarp<RV, LMAX>& lw, const LatRow<LMAX>& rt, const double (&pv)[RV],
                                              const double (&ps)[RV], double (&ap)[RV], double (&atps)[RV]) {
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        lw.X[j * 32 + lw.lane] = pv[j];
        lw.X[lw.P + 16 + j * 32 + lw.lane] = ps[j];
    }
    if (lw.lane == 0) *lw.ctrl = kLatPair;
    lat_bar_a(lw.T);
    const double s0 = lat_row<LMAX>(lw.ra, lw.xaddr, lw.nsteps);
    const double s1 = lat_row<LMAX>(rt, lw.xaddr, lw.nsteps);
    if (lw.srow >= 0) {
        lw.Y[lw.srow] = s0;
        lw.Y[lw.P + lw.srow] = s1;
    }
    lat_bar_b(lw.T);
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        ap[j] = lw.Y[j * 32 + lw.lane];
        atps[j] = lw.Y[lw.P + j * 32 + lw.lane];
    }
}

// Warps 1..: compute their rows of every SpMV the leader posts until it posts kLatExit.
template <int RV, int LMAX, int ALGO>
__device__ __forceinline__ void lat_helper(LatWarp<RV, LMAX>& lw, const LatRow<(ALGO == kBiCG ? LMAX : 1)>& rt) {
    for (;;) {
        lat_bar_a(lw.T);
        const int op = *lw.ctrl;
        if (op == kLatExit) return;
        const double s0 = lat_row<LMAX>(lw.ra, lw.xaddr, lw.nsteps);
        if constexpr (ALGO == kBiCG) {
            if (op == kLatPair) {
                const double s1 = lat_row<LMAX>(rt, lw.xaddr, lw.nsteps);
                if (lw.srow >= 0) lw.Y[lw.P + lw.srow] = s1;
            }
        }
        if (lw.srow >= 0) lw.Y[lw.srow] = s0;
        lat_bar_b(lw.T);
    }
}

template <int R, int RV, int LMAX>
__device__ __forceinline__ double lat_fresh_rms(LatWarp<RV, LMAX>& lw, const double (&x)[RV], const double (&b)[RV],
                                                int n) {
    double ax[RV];
    lat_spmv(lw, x, ax);
    double sq[1][RV];
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        const double ri = dsub(b[j], ax[j]);
        sq[0][j] = dmul(ri, ri);
    }
    double o[1];
    tmem_reduce<1, R, RV>(sq, o);
    return __dsqrt_rn(ddiv(o[0], static_cast<double>(n)));
}

template <int R, int RV, int LMAX, int ALGO>
__global__ void __launch_bounds__(RV * 32, 1) block_cells_latency_kernel(const LatencyParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int t = threadIdx.x, T = blockDim.x, lane = t % 32, w = t / 32;
    __shared__ int s_ctrl;
    double* Y = reinterpret_cast<double*>(smem);  // [2][P]
    LatWarp<RV, LMAX> lw;
    lw.P = p.P;
    lw.T = T;
    lw.lane = lane;
    lw.Y = Y;
    lw.X = Y + 2 * p.P;
    lw.xaddr = static_cast<uint32_t>(__cvta_generic_to_shared(lw.X));
    lw.srow = p.rowof[t];
    lw.nsteps = p.steps[t];
    lw.ctrl = &s_ctrl;
    // Y slots >= n, the zero slots and rows >= n of the gather region: +0.0 for good
    for (int i = t; i < 2 * p.P + p.xs; i += T) Y[i] = 0.0;
#pragma unroll
    for (int e = 0; e < LMAX; ++e) lw.ra.o[e] = p.rxo[e * T + t];
    LatRow<(ALGO == kBiCG ? LMAX : 1)> rt;
    if constexpr (ALGO == kBiCG) {
#pragma unroll
        for (int e = 0; e < LMAX; ++e) rt.o[e] = p.txo[e * T + t];
    }
    const double smax = p.sigma_max;

    for (int gl = blockIdx.x; gl < p.group_count; gl += gridDim.x) {
        if (p.gate.ready && t == 0) gate_wait(p.gate, gl);
        __syncthreads();  // also: the previous group's last reads of X / Y are done
        const int64_t cell0 = p.cell_offset + static_cast<int64_t>(gl) * p.kc;
        const double* src = p.values + cell0 * p.nnz;
        const double* bsrc = p.rhs + cell0 * p.species;
#pragma unroll
        for (int e = 0; e < LMAX; ++e) {
            const int vi = p.rvi[e * T + t];
            lw.ra.a[e] = vi >= 0 ? __ldg(src + vi) : 0.0;
        }
        if constexpr (ALGO == kBiCG) {
#pragma unroll
            for (int e = 0; e < LMAX; ++e) {
                const int vi = p.tvi[e * T + t];
                rt.a[e] = vi >= 0 ? __ldg(src + vi) : 0.0;
            }
        }
        if (w != 0) {  // helper warps: their rows of every SpMV of this group
            lat_helper<RV, LMAX, ALGO>(lw, rt);
            continue;
        }
        double b[RV], x[RV];
#pragma unroll
        for (int j = 0; j < RV; ++j) {
            const int row = j * 32 + lane;
            b[j] = row < p.n ? __ldg(bsrc + row) : 0.0;
            x[j] = 0.0;
        }
        double fres = 0.0;
        int iters = 0;
        bool conv = false, brk = false;
        if constexpr (ALGO == kBiCGStab) {
            double dinv[RV];
#pragma unroll
            for (int j = 0; j < RV; ++j) {
                const int row = j * 32 + lane;
                const int di = row < p.n ? p.didx[row] : -1;
                const double d = di >= 0 ? __ldg(src + di) : 0.0;
                dinv[j] = row < p.n ? (d != 0.0 ? ddiv(1.0, d) : 1.0) : 0.0;
            }
            double r[RV], rh[RV], pv[RV], v[RV];
            {
                double ax[RV];
                lat_spmv(lw, x, ax);
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    r[j] = dadd(b[j], -ax[j]);  // 1*b + (-1)*Ax; rows >= n: 0 + -0 = +0
                    rh[j] = r[j];
                    pv[j] = 0.0;
                    v[j] = 0.0;
                }
            }
            double sigma, rho_next;
            {
                double q[2][RV], o[2];
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    q[0][j] = dmul(r[j], r[j]);
                    q[1][j] = dmul(rh[j], r[j]);
                }
                tmem_reduce<2, R, RV>(q, o);
                sigma = o[0];
                rho_next = o[1];
            }
            if (sigma <= smax) {
                fres = lat_fresh_rms<R>(lw, x, b, p.n);
                conv = fres <= p.tol;
            }
            if (!conv) {
                double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
                double aw = ddiv(alpha, omega);  // alpha/omega of beta, computed as soon as omega is known
                double pt[RV];  // p - omega v of the next p update, formed as soon as omega is known
#pragma unroll
                for (int j = 0; j < RV; ++j) pt[j] = dsub(pv[j], dmul(omega, v[j]));
#ifdef BC_LAT_PROFILE
                long long prof_t = clock64(), prof_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
                for (int it = 1; it <= p.max_iter; ++it) {
                    const double rho = rho_next;
                    if (scalar_breaks(rho)) { brk = true; break; }
                    const double beta = dmul(ddiv(rho, rho_prev), aw);
                    double y[RV];
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        pv[j] = dadd(r[j], dmul(beta, pt[j]));
                        y[j] = dmul(dinv[j], pv[j]);
                    }
                    LAT_MARK(0);
                    lat_spmv(lw, y, v);
                    LAT_MARK(1);
                    double den;
                    {
                        double q[1][RV], o[1];
#pragma unroll
                        for (int j = 0; j < RV; ++j) q[0][j] = dmul(rh[j], v[j]);
                        tmem_reduce<1, R, RV>(q, o);
                        den = o[0];
                    }
                    LAT_MARK(2);
                    if (scalar_breaks(den)) { brk = true; break; }
                    alpha = ddiv(rho, den);
                    double z[RV];
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        r[j] = dsub(r[j], dmul(alpha, v[j]));  // r now holds s
                        z[j] = dmul(dinv[j], r[j]);
                        x[j] = dadd(x[j], dmul(alpha, y[j]));
                    }
                    LAT_MARK(3);
                    double tv[RV];
                    lat_spmv(lw, z, tv);
                    LAT_MARK(4);
                    double tt, ts;
                    {
                        double q[2][RV], o[2];
#pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(tv[j], tv[j]);
                            q[1][j] = dmul(tv[j], r[j]);
                        }
                        tmem_reduce<2, R, RV>(q, o);
                        tt = o[0];
                        ts = o[1];
                    }
                    LAT_MARK(5);
                    if (tt != 0.0 && scalar_breaks(tt)) { brk = true; break; }
                    omega = tt == 0.0 ? 0.0 : ddiv(ts, tt);
                    aw = ddiv(alpha, omega);  // next beta's factor, off the critical path
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        x[j] = dadd(x[j], dmul(omega, z[j]));
                        r[j] = dsub(r[j], dmul(omega, tv[j]));
                        pt[j] = dsub(pv[j], dmul(omega, v[j]));  // the next p update's inner term
                    }
                    rho_prev = rho;
                    iters = it;
                    LAT_MARK(6);
                    {
                        double q[2][RV], o[2];
#pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(r[j], r[j]);
                            q[1][j] = dmul(rh[j], r[j]);
                        }
                        tmem_reduce<2, R, RV>(q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    LAT_MARK(7);
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (sigma <= smax) {
                        const double f = lat_fresh_rms<R>(lw, x, b, p.n);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                    if (scalar_breaks(omega)) { brk = true; break; }
                    LAT_MARK(8);
                }
#ifdef BC_LAT_PROFILE
                if (blockIdx.x == 0 && t == 0)
                    for (int i = 0; i < 9; ++i) bc_lat_prof[i] += prof_acc[i];
#endif
                if (!conv) {
                    fres = lat_fresh_rms<R>(lw, x, b, p.n);
                    conv = !brk && fres <= p.tol;
                }
            }
        } else {
            // BiCG, bicg.cpp:42-142 operation for operation (as bc_tmem.cuh's kBiCG)
            double r[RV], rs[RV], pv[RV], ps[RV];
            {
                double ax[RV];
                lat_spmv(lw, x, ax);
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    r[j] = dadd(b[j], -ax[j]);
                    rs[j] = r[j];
                    pv[j] = r[j];
                    ps[j] = r[j];
                }
            }
            double sigma, rho_next;
            {
                double q[2][RV], o[2];
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    q[0][j] = dmul(r[j], r[j]);
                    q[1][j] = dmul(rs[j], r[j]);
                }
                tmem_reduce<2, R, RV>(q, o);
                sigma = o[0];
                rho_next = o[1];
            }
            if (sigma <= smax) {
                fres = lat_fresh_rms<R>(lw, x, b, p.n);
                conv = fres <= p.tol;
            }
            if (!conv) {
                double rho_prev = 0.0;
                for (int it = 1; it <= p.max_iter; ++it) {
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
                    lat_spmv_pair(lw, rt, pv, ps, ap, atps);
                    double den;
                    {
                        double q[1][RV], o[1];
#pragma unroll
                        for (int j = 0; j < RV; ++j) q[0][j] = dmul(ps[j], ap[j]);
                        tmem_reduce<1, R, RV>(q, o);
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
                    {
                        double q[2][RV], o[2];
#pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(r[j], r[j]);
                            q[1][j] = dmul(rs[j], r[j]);
                        }
                        tmem_reduce<2, R, RV>(q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (sigma <= smax) {
                        const double f = lat_fresh_rms<R>(lw, x, b, p.n);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                }
                if (!conv) {
                    fres = lat_fresh_rms<R>(lw, x, b, p.n);
                    conv = !brk && fres <= p.tol;
                }
            }
        }
        if (lane == 0) s_ctrl = kLatExit;  // release the helpers
        lat_bar_a(T);
        {
            double* xdst = p.x_out + cell0 * p.species;
#pragma unroll
            for (int j = 0; j < RV; ++j)
                if (j * 32 + lane < p.n) xdst[j * 32 + lane] = x[j];
            if (lane == 0) {
                const int64_t g = p.group_offset + gl;
                p.g_iters[g] = iters;
                p.g_rms[g] = fres;
                p.g_flags[g] = static_cast<uint8_t>((conv ? 1 : 0) | (brk ? 2 : 0));
            }
        }
    }
}

}  // namespace bc
