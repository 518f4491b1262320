// bc_tmem.cuh -- Block-cells(1) Jacobi-BiCGSTAB with the SpMV operands in
// Tensor Memory (the B200 hot path; K1 v2).
//
// The v1 kernel (bc_block.cuh) is bound by shared-memory wavefronts: per SpMV
// step a lane loads its schedule word (1 wavefront), its matrix value (2) and
// the gathered vector entry (~3.7 after placement), plus row-end stores.
// TMEM (256 KB/SM, read with tcgen05.ld on its own datapath -- measured to
// overlap completely with LDS traffic, tools/microbench.py) takes the first
// two off the shared-memory pipe:
//
//   TMEM lane 32q+L, columns [0, S8)            schedule word of step t for lane L
//                                               (one copy per lane quarter q, shared
//                                               by the quarter's warps)
//   TMEM lane 32q+L, columns [S8 + 2*S8*s, ...) value of step t for lane L of the
//                                               cell held by warp (q, s), fp64 as
//                                               two 32-bit columns
//
// Every step's column address is warp-uniform, which is exactly the
// tcgen05.ld.32x32b shape (each thread reads its own lane).  A CTA is 16 warps
// (4 per lane quarter), owns all 512 columns, and stays resident (one per SM);
// each warp solves one cell at a time, fetched from an atomic counter.
// Arithmetic, schedule order and reductions are those of bc_block.cuh, so the
// results are bit-identical to v1 and to the oracle.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bc_block.cuh"

namespace bc {

struct TmemParams {
    const double* values;  // cells * nnz
    const double* rhs;     // cells * species
    double* x_out;
    int32_t* g_iters;
    double* g_rms;
    uint8_t* g_flags;
    const uint32_t* words;  // S * 32 (A schedule)
    const int32_t* vidx;    // S * 32: schedule slot -> value index in the cell
    const int32_t* didx;    // species: value index of the diagonal, -1 if none
    const int32_t* xpos;    // species: gather slot of each row
    unsigned int* counter;
    int64_t cell_offset, group_offset;
    int group_count;
    int n, nnz, S, S8, P;
    int species, kc;        // group = kc cells of `species` rows
    int xslots;             // shared doubles of the gather vector (multiple of 32)
    int cells_per_quarter;  // warps per lane quarter
    double tol;
    int64_t max_iter;
};

__device__ __forceinline__ void tm_ld_x8(uint32_t addr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
}
__device__ __forceinline__ void tm_ld_x16(uint32_t addr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
__device__ __forceinline__ void tm_st_x8(uint32_t addr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(addr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// y = A x: publish x at its gather slots, walk the TMEM-resident schedule
// (8 steps per tcgen05.ld pair), results through the shared Y vector.
template <int R, int RV>
__device__ __forceinline__ void tmem_spmv(const Ctx<1, R, RV>& c, uint32_t wcol, uint32_t vcol, int S8,
                                          const double (&x)[RV], double (&y)[RV]) {
#pragma unroll
    for (int j = 0; j < RV; ++j)
        if (c.valid(j)) c.Xs[c.xa[j]] = x[j];
    __syncwarp();
    double acc = 0.0;
    for (int t0 = 0; t0 < S8; t0 += 8) {
        uint32_t w[8], v[16];
        tm_ld_x8(wcol + t0, w);
        tm_ld_x16(vcol + 2 * t0, v);
        tm_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double a = __hiloint2double(static_cast<int>(v[2 * u + 1]), static_cast<int>(v[2 * u]));
            const double xv = c.Xs[w[u] & kColMask];
            acc = dadd(acc, dmul(a, xv));
            if (w[u] & kEndBit) {
                c.Ys[(w[u] >> kColBits) & kColMask] = acc;
                acc = 0.0;
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < RV; ++j) y[j] = c.valid(j) ? c.Ys[c.row(j)] : 0.0;
}

template <int R, int RV>
__device__ __forceinline__ double tmem_fresh_rms(const Ctx<1, R, RV>& cc, uint32_t wcol, uint32_t vcol, int S8,
                                                 const double (&x)[RV], const double* bsrc) {
    Ctx<1, R, RV> c = cc;
    double ax[RV];
    tmem_spmv(c, wcol, vcol, S8, x, ax);
    double sq[1][RV];
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        const double bj = c.valid(j) ? bsrc[c.row(j)] : 0.0;
        const double ri = dsub(bj, ax[j]);
        sq[0][j] = dmul(ri, ri);
    }
    double out[1];
    team_reduce<1>(c, sq, out);
    return __dsqrt_rn(ddiv(out[0], static_cast<double>(c.n)));
}

template <int R, int RV>
__global__ void __launch_bounds__(512, 1) block_cells_tmem_kernel(const TmemParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_taddr;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int quarter = warp % 4, slot = warp / 4;
    int32_t* s_vidx = reinterpret_cast<int32_t*>(smem);                         // S8*32
    double* s_vec = reinterpret_cast<double*>(smem + sizeof(int32_t) * p.S8 * 32);  // per warp: X | Y

    for (int i = threadIdx.x; i < p.S8 * 32; i += blockDim.x) s_vidx[i] = i < p.S * 32 ? p.vidx[i] : 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&s_taddr))),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t lane_base = s_taddr + (static_cast<uint32_t>(32 * quarter) << 16);
    const uint32_t wcol = lane_base;                                        // words: columns [0, S8)
    const uint32_t vcol = lane_base + p.S8 + 2u * p.S8 * static_cast<uint32_t>(slot);
    // words into TMEM, once per quarter (schedule is the same for every cell)
    if (slot == 0) {
        for (int t0 = 0; t0 < p.S8; t0 += 8) {
            uint32_t w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = (t0 + u < p.S) ? p.words[(t0 + u) * 32 + lane] : 0u;
            tm_st_x8(wcol + t0, w);
        }
        tm_wait_st();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    const bool active = slot < p.cells_per_quarter;
    Ctx<1, R, RV> c;
    c.tm.id = warp;
    c.tm.tid = lane;
    c.tm.w = 0;
    c.tm.lane = lane;
    c.n = p.n;
    c.P = p.P;
    c.Xs = s_vec + static_cast<size_t>(warp) * (p.xslots + ((p.n + 31) & ~31));
    c.Ys = c.Xs + p.xslots;
#pragma unroll
    for (int j = 0; j < RV; ++j) c.xa[j] = c.valid(j) ? p.xpos[c.row(j)] : 0;
    const double nd = static_cast<double>(p.n);

    while (active) {
        unsigned int gv = 0;
        if (lane == 0) gv = atomicAdd(p.counter, 1u);
        const int gl = static_cast<int>(__shfl_sync(0xffffffffu, gv, 0));
        if (gl >= p.group_count) break;
        const int64_t cell0 = p.cell_offset + static_cast<int64_t>(gl) * p.kc;
        const double* src = p.values + cell0 * p.nnz;
        const double* bsrc = p.rhs + cell0 * p.species;

        // stage this cell's values into TMEM in schedule order (once per solve)
        for (int t0 = 0; t0 < p.S8; t0 += 4) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double a = __ldg(src + s_vidx[(t0 + u) * 32 + lane]);
                v[2 * u] = static_cast<uint32_t>(__double2loint(a));
                v[2 * u + 1] = static_cast<uint32_t>(__double2hiint(a));
            }
            tm_st_x8(vcol + 2 * t0, v);
        }
        for (int i = lane; i < p.n; i += 32) c.Ys[i] = 0.0;  // empty rows read +0.0
        tm_wait_st();
        __syncwarp();

        double x[RV], dinv[RV];
#pragma unroll
        for (int j = 0; j < RV; ++j) {
            x[j] = 0.0;
            double d = 0.0;
            if (c.valid(j)) {
                const int di = p.didx[c.row(j)];
                d = di >= 0 ? __ldg(src + di) : 0.0;
                dinv[j] = d != 0.0 ? ddiv(1.0, d) : 1.0;
            } else {
                dinv[j] = 0.0;
            }
        }
        int64_t iters = 0;
        bool conv = false, brk = false;
        double fres = 0.0;
        double r[RV], rh[RV], pv[RV], v[RV];
        {
            double ax[RV];
            tmem_spmv(c, wcol, vcol, p.S8, x, ax);
#pragma unroll
            for (int j = 0; j < RV; ++j) {
                const double bj = c.valid(j) ? __ldcs(bsrc + c.row(j)) : 0.0;
                r[j] = c.valid(j) ? dadd(bj, -ax[j]) : 0.0;  // 1*b + (-1)*Ax
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
            fres = tmem_fresh_rms(c, wcol, vcol, p.S8, x, bsrc);
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
                tmem_spmv(c, wcol, vcol, p.S8, y, v);
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
                double z[RV];
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    r[j] = dsub(r[j], dmul(alpha, v[j]));          // r now holds s
                    z[j] = dmul(dinv[j], r[j]);
                    x[j] = dadd(x[j], dmul(alpha, dmul(dinv[j], pv[j])));  // y = dinv*p recomputed
                }
                double t[RV];
                tmem_spmv(c, wcol, vcol, p.S8, z, t);
                double tt, ts;
                {
                    double q[2][RV], o[2];
#pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        q[0][j] = dmul(t[j], t[j]);
                        q[1][j] = dmul(t[j], r[j]);
                    }
                    team_reduce<2>(c, q, o);
                    tt = o[0];
                    ts = o[1];
                }
                if (tt != 0.0 && scalar_breaks(tt)) { brk = true; break; }
                omega = tt == 0.0 ? 0.0 : ddiv(ts, tt);
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    x[j] = dadd(x[j], dmul(omega, dmul(dinv[j], r[j])));  // z = dinv*s recomputed
                    r[j] = dsub(r[j], dmul(omega, t[j]));
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
                    const double f = tmem_fresh_rms(c, wcol, vcol, p.S8, x, bsrc);
                    if (f <= p.tol) {
                        fres = f;
                        conv = true;
                        break;
                    }
                }
                if (scalar_breaks(omega)) { brk = true; break; }
            }
            if (!conv) {
                fres = tmem_fresh_rms(c, wcol, vcol, p.S8, x, bsrc);
                conv = !brk && fres <= p.tol;
            }
        }
        double* xdst = p.x_out + cell0 * p.species;
#pragma unroll
        for (int j = 0; j < RV; ++j)
            if (c.valid(j)) xdst[c.row(j)] = x[j];
        if (lane == 0) {
            const int64_t g = p.group_offset + gl;
            p.g_iters[g] = static_cast<int32_t>(iters);
            p.g_rms[g] = fres;
            p.g_flags[g] = static_cast<uint8_t>((conv ? 1 : 0) | (brk ? 2 : 0));
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "r"(512));
}

}  // namespace bc
