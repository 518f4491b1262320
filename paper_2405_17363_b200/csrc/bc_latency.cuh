// bc_latency.cuh -- latency mode for small batches (BASELINE configs[0]: 100
// cells; the tail of a partial wave): one CTA of W = P/32 warps per group,
// one thread per row.
//
// The throughput kernel (bc_tmem.cuh) packs a cell's 1556 entries onto one
// warp (52 schedule steps per SpMV) and overlaps 16 cells per SM to fill the
// shared-memory pipe; alone on an SM one cell takes ~4.5 ms for 1000
// iterations (~8,900 cycles per iteration, a dependent-latency chain).  When
// there are fewer groups than SMs can overlap, latency is the metric, so this
// kernel spreads a group over P = next_pow2(n) threads, the geometry of the
// reference's own Block-cells launch (one thread per row, exec_model.cpp:
// 115-122, 134-158):
//
//   * thread t owns row t (t < n) -- exactly the slot of the reduction tree
//     (team_reduce with R = 1: cross-warp levels through shared memory, then
//     the xor butterfly), so the SpMV result needs no exchange: the row's sum
//     is computed by the thread that owns it;
//   * thread t keeps row t's values (CSR order) and gather offsets in
//     registers, padded to LMAX with (0.0, the always-zero slot): the padding
//     adds exact +0.0 to a sum that started at +0.0 and is therefore never
//     -0.0, so every thread runs LMAX unconditional steps and the result is
//     the reference's row sum (csr.cpp:90-101) bit for bit;
//   * BiCG's A^T row t (column t of A, ascending source row, csr.cpp:129-142)
//     runs beside it as a second independent chain over the p~ copy;
//   * per SpMV: one store of the thread's entry of the vector, one barrier,
//     LMAX gathers + the ordered multiply-add chain; per reduction: one store,
//     one barrier, W loads and the butterfly (double-buffered partials).
// The arithmetic is the TMEM kernel's / the oracle's, operation for
// operation, with rows >= n carrying exact +0.0 (dinv 0, values 0).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bc_block.cuh"

namespace bc {

struct LatencyParams {
    const double* values;  // cells * nnz
    const double* rhs;     // cells * species
    double* x_out;
    int32_t* g_iters;
    double* g_rms;
    uint8_t* g_flags;
    const int32_t* rvi;    // [lmax][P]: group value index of row t's e-th entry, -1 = padding
    const uint16_t* rxo;   // [lmax][P]: byte offset of its gather slot (padding: the zero slot)
    const int32_t* tvi;    // BiCG: [lmaxt][P], column t's entries in ascending row order
    const uint16_t* txo;   // BiCG: byte offsets into the p~ copy
    const int32_t* didx;   // n: group value index of the diagonal, -1 if none
    int64_t cell_offset, group_offset;
    int group_count;
    int n, nnz, P, species, kc;
    int xslots;            // doubles of the gather region (p, zero slot, [p~])
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

// y_t = sum_e a[e] * X[o[e]] in CSR order from +0.0 (gathers issued first).
template <int LMAX>
__device__ __forceinline__ double lat_row(const LatRow<LMAX>& rw, uint32_t xbase) {
    double g[LMAX];
#pragma unroll
    for (int e = 0; e < LMAX; ++e) g[e] = lds64(xbase + rw.o[e]);
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < LMAX; ++e) acc = dadd(acc, dmul(rw.a[e], g[e]));
    return acc;
}

template <int W, int LMAX>
__device__ __forceinline__ double lat_spmv(const Team<W>& tm, double* X, uint32_t xbase, int t, double v,
                                           const LatRow<LMAX>& rw) {
    X[t] = v;
    tm.sync();
    return lat_row<LMAX>(rw, xbase);
}

template <int W, int LMAX>
__device__ __forceinline__ double lat_fresh_rms(Ctx<W, 1, 1>& c, double* X, uint32_t xbase, int t, double x,
                                                double b, const LatRow<LMAX>& rw) {
    const double ax = lat_spmv<W, LMAX>(c.tm, X, xbase, t, x, rw);
    const double ri = dsub(b, ax);
    double q[1][1] = {{dmul(ri, ri)}}, o[1];
    team_reduce<1>(c, q, o);
    return __dsqrt_rn(ddiv(o[0], static_cast<double>(c.n)));
}

template <int W, int LMAX, int ALGO>
__global__ void __launch_bounds__(W * 32, 1) block_cells_latency_kernel(const LatencyParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* X = reinterpret_cast<double*>(smem);                 // xslots doubles
    double* red = X + p.xslots;                                  // [2][4][W][32]
    const uint32_t xbase = static_cast<uint32_t>(__cvta_generic_to_shared(X));
    const int t = threadIdx.x;
    const bool valid = t < p.n;
    Ctx<W, 1, 1> c;
    c.tm.id = 0;
    c.tm.w = t / 32;
    c.tm.lane = t % 32;
    c.tm.tid = t;
    c.n = p.n;
    c.P = p.P;
    c.red = red;
    c.red_buf = 0;
    for (int i = t; i < p.xslots; i += W * 32) X[i] = 0.0;  // the zero slot(s) stay +0.0
    LatRow<LMAX> ra;
    LatRow<(ALGO == kBiCG ? LMAX : 1)> rt;
#pragma unroll
    for (int e = 0; e < LMAX; ++e) ra.o[e] = p.rxo[e * p.P + t];
    if constexpr (ALGO == kBiCG) {
#pragma unroll
        for (int e = 0; e < LMAX; ++e) rt.o[e] = p.txo[e * p.P + t];
    }
    const double smax = p.sigma_max;

    for (int gl = blockIdx.x; gl < p.group_count; gl += gridDim.x) {
        if (p.gate.ready) {
            if (t == 0) gate_wait(p.gate, gl);
        }
        c.tm.sync();  // also: the previous group's last reads of X / red are done
        const int64_t cell0 = p.cell_offset + static_cast<int64_t>(gl) * p.kc;
        const double* src = p.values + cell0 * p.nnz;
        const double* bsrc = p.rhs + cell0 * p.species;
#pragma unroll
        for (int e = 0; e < LMAX; ++e) {
            const int vi = p.rvi[e * p.P + t];
            ra.a[e] = vi >= 0 ? __ldg(src + vi) : 0.0;
        }
        if constexpr (ALGO == kBiCG) {
#pragma unroll
            for (int e = 0; e < LMAX; ++e) {
                const int vi = p.tvi[e * p.P + t];
                rt.a[e] = vi >= 0 ? __ldg(src + vi) : 0.0;
            }
        }
        const double b = valid ? __ldg(bsrc + t) : 0.0;
        double x = 0.0, fres = 0.0;
        int iters = 0;
        bool conv = false, brk = false;
        if constexpr (ALGO == kBiCGStab) {
            double dinv = 0.0;
            if (valid) {
                const int di = p.didx[t];
                const double d = di >= 0 ? __ldg(src + di) : 0.0;
                dinv = d != 0.0 ? ddiv(1.0, d) : 1.0;
            }
            const double ax = lat_spmv<W, LMAX>(c.tm, X, xbase, t, x, ra);
            double r = dadd(b, -ax);  // 1*b + (-1)*Ax; rows >= n: 0 + -0 = +0
            const double rh = r;
            double pv = 0.0, v = 0.0;
            double sigma, rho_next;
            {
                double q[2][1] = {{dmul(r, r)}, {dmul(rh, r)}}, o[2];
                team_reduce<2>(c, q, o);
                sigma = o[0];
                rho_next = o[1];
            }
            if (sigma <= smax) {
                fres = lat_fresh_rms<W, LMAX>(c, X, xbase, t, x, b, ra);
                conv = fres <= p.tol;
            }
            if (!conv) {
                double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
                for (int it = 1; it <= p.max_iter; ++it) {
                    const double rho = rho_next;
                    if (scalar_breaks(rho)) { brk = true; break; }
                    const double beta = dmul(ddiv(rho, rho_prev), ddiv(alpha, omega));
                    pv = dadd(r, dmul(beta, dsub(pv, dmul(omega, v))));
                    const double y = dmul(dinv, pv);
                    v = lat_spmv<W, LMAX>(c.tm, X, xbase, t, y, ra);
                    double den;
                    {
                        double q[1][1] = {{dmul(rh, v)}}, o[1];
                        team_reduce<1>(c, q, o);
                        den = o[0];
                    }
                    if (scalar_breaks(den)) { brk = true; break; }
                    alpha = ddiv(rho, den);
                    r = dsub(r, dmul(alpha, v));  // r now holds s
                    const double z = dmul(dinv, r);
                    x = dadd(x, dmul(alpha, y));
                    const double tv = lat_spmv<W, LMAX>(c.tm, X, xbase, t, z, ra);
                    double tt, ts;
                    {
                        double q[2][1] = {{dmul(tv, tv)}, {dmul(tv, r)}}, o[2];
                        team_reduce<2>(c, q, o);
                        tt = o[0];
                        ts = o[1];
                    }
                    if (tt != 0.0 && scalar_breaks(tt)) { brk = true; break; }
                    omega = tt == 0.0 ? 0.0 : ddiv(ts, tt);
                    x = dadd(x, dmul(omega, z));
                    r = dsub(r, dmul(omega, tv));
                    rho_prev = rho;
                    iters = it;
                    {
                        double q[2][1] = {{dmul(r, r)}, {dmul(rh, r)}}, o[2];
                        team_reduce<2>(c, q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (sigma <= smax) {
                        const double f = lat_fresh_rms<W, LMAX>(c, X, xbase, t, x, b, ra);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                    if (scalar_breaks(omega)) { brk = true; break; }
                }
                if (!conv) {
                    fres = lat_fresh_rms<W, LMAX>(c, X, xbase, t, x, b, ra);
                    conv = !brk && fres <= p.tol;
                }
            }
        } else {
            // BiCG, bicg.cpp:42-142 operation for operation; A p on the p copy
            // (slots [0, P)) and A^T p~ on the p~ copy (slots [P + 1, 2P + 1)),
            // one barrier for both
            const double ax = lat_spmv<W, LMAX>(c.tm, X, xbase, t, x, ra);
            double r = dadd(b, -ax);
            double rs = r, pv = r, ps = r;
            double sigma, rho_next;
            {
                double q[2][1] = {{dmul(r, r)}, {dmul(rs, r)}}, o[2];
                team_reduce<2>(c, q, o);
                sigma = o[0];
                rho_next = o[1];
            }
            if (sigma <= smax) {
                fres = lat_fresh_rms<W, LMAX>(c, X, xbase, t, x, b, ra);
                conv = fres <= p.tol;
            }
            if (!conv) {
                double rho_prev = 0.0;
                for (int it = 1; it <= p.max_iter; ++it) {
                    const double rho = rho_next;
                    if (scalar_breaks(rho)) { brk = true; break; }
                    if (it > 1) {
                        const double beta = ddiv(rho, rho_prev);
                        pv = dadd(r, dmul(beta, pv));
                        ps = dadd(rs, dmul(beta, ps));
                    }
                    X[t] = pv;
                    X[p.P + 1 + t] = ps;
                    c.tm.sync();
                    const double ap = lat_row<LMAX>(ra, xbase);
                    const double atps = lat_row<LMAX>(rt, xbase);
                    double den;
                    {
                        double q[1][1] = {{dmul(ps, ap)}}, o[1];
                        team_reduce<1>(c, q, o);
                        den = o[0];
                    }
                    if (scalar_breaks(den)) { brk = true; break; }
                    const double alpha = ddiv(rho, den);
                    const double nalpha = -alpha;
                    x = dadd(x, dmul(alpha, pv));
                    r = dadd(r, dmul(nalpha, ap));
                    rs = dadd(rs, dmul(nalpha, atps));
                    rho_prev = rho;
                    iters = it;
                    {
                        double q[2][1] = {{dmul(r, r)}, {dmul(rs, r)}}, o[2];
                        team_reduce<2>(c, q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (sigma <= smax) {
                        const double f = lat_fresh_rms<W, LMAX>(c, X, xbase, t, x, b, ra);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                }
                if (!conv) {
                    fres = lat_fresh_rms<W, LMAX>(c, X, xbase, t, x, b, ra);
                    conv = !brk && fres <= p.tol;
                }
            }
        }
        if (valid) p.x_out[cell0 * p.species + t] = x;
        if (t == 0) {
            const int64_t g = p.group_offset + gl;
            p.g_iters[g] = iters;
            p.g_rms[g] = fres;
            p.g_flags[g] = static_cast<uint8_t>((conv ? 1 : 0) | (brk ? 2 : 0));
        }
    }
}

}  // namespace bc
