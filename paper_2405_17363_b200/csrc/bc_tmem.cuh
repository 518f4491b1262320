// bc_tmem.cuh -- the B200 hot path (K1 v3): Block-cells solves of one cell (or
// any group whose reduction tree has <= 16 slots per lane) per warp or per
// team of 2/4 warps, BiCG or Jacobi-BiCGSTAB, with the SpMV operands in
// Tensor Memory.
//
// The v1 kernel (bc_block.cuh) is bound by shared-memory wavefronts: per SpMV
// step a lane loads its schedule word (1 wavefront), its matrix value (2) and
// the gathered vector entry (~3.7), plus row-end stores.  TMEM (256 KB/SM,
// read with tcgen05.ld on its own datapath -- measured to overlap completely
// with LDS traffic, tools/microbench.py) takes the first two off the shared-
// memory pipe:
//
//   TMEM lane 32q+L, columns [0, S/2)      16-bit schedule words of lane L
//                                          (team role q % W), two steps per
//                                          column, shared by the quarter's warps
//   then per warp (q, s): 2S columns       fp64 values of lane L's steps for the
//                                          group it holds; BiCGSTAB adds 2*RV
//                                          columns of D^-1
//
// Every column address is warp-uniform -- exactly the tcgen05.ld.32x32b shape
// (each thread reads its own lane).  A CTA owns all 512 columns and stays
// resident (one per SM); each warp (team) solves one group at a time, fetched
// from an atomic counter.  The schedule (bc_plan.hpp TmemSchedule,
// bc_tmem_plan.cpp) pads rows to even length with zero entries and runs two
// rows per lane at a time (stream 0 on even steps, stream 1 on odd), so row
// ends are tested once per two steps with the flag riding in an address word;
// lane L's k-th row of stream s goes to Y[s*ystream + k*32W + L]; the gathered
// vector is kept in two placements (identity, and rotated per 16 columns) so
// gathers almost never conflict and publishes never do.  BiCG's pair schedule
// puts A's rows on stream 0 and A^T's on stream 1: both products in one pass.
//
// Rows beyond n (register slots of the padded reduction tree) carry exact
// +0.0 through every update -- 0-(+-0) = +0, 0+(+-0) = +0, 0*0 = +0 -- so the
// arithmetic needs no validity tests: those rows publish into a trash slot and
// read the always-zero Y slot.  The convergence test sqrt(sigma/n) <= tol is
// evaluated as sigma <= sigma_max with sigma_max computed on the host as the
// largest double satisfying it (sqrt and / are correctly rounded and
// monotone, so the two tests agree for every sigma, NaN included).
// Arithmetic order and reductions are those of bc_block.cuh and the oracle:
// results are bit-identical.
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
    const uint16_t* words;  // S * 32: gather byte offset | end << 15
    const int32_t* vidx;    // S * 32: group value index, -1 = padding (0.0)
    const int32_t* didx;    // n: group value index of the diagonal, -1 if none
    const uint32_t* lane_xy;  // RV * 32: copy-0 gather slot | Y slot << 16 per (slot j, lane)
    const uint32_t* lane_x1;  // ((RV+1)/2) * 32: copy-1 gather slots, two row slots per word
    const uint32_t* lane_xyT; // BiCG pair schedules: the same two tables for p~ / A^T p~
    const uint32_t* lane_x1T;
    unsigned int* counter;
    int64_t cell_offset, group_offset;
    int group_count;
    int n, nnz, S, P;
    int species, kc;        // group = kc cells of `species` rows
    int xslots, yslots;     // shared doubles per warp: X | Y (multiples of 32)
    int xalign;             // bytes per warp X region: a power of two >= 8 * xslots
    int ystream;            // Y slots per row stream (TmemSchedule::ystream)
    int cells_per_quarter;  // warps per lane quarter
    double sigma_max;       // sqrt(sigma/n) <= tol  <=>  sigma <= sigma_max
    double tol;             // the fresh-residual test keeps the literal comparison
    int max_iter;
    InputGate gate;         // streamed host inputs (bc_solve), or gate.ready == nullptr
};

__device__ __forceinline__ void tm_ld_x2(uint32_t addr, uint32_t (&r)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ void tm_ld_x8(uint32_t addr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
}
__device__ __forceinline__ void tm_st_x2(uint32_t addr, const uint32_t (&r)[2]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(addr), "r"(r[0]), "r"(r[1])
                 : "memory");
}
__device__ __forceinline__ void tm_st_x8(uint32_t addr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(addr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void tm_ld_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void tm_ld_x16(uint32_t addr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}

// A per-lane vector of RV doubles in TMEM (two 32-bit columns each): the
// Jacobi scaling D^-1 lives there rather than in registers.
template <int RV>
__device__ __forceinline__ void tm_store_vec(uint32_t col, const double (&v)[RV]) {
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        const uint32_t w[2] = {static_cast<uint32_t>(__double2loint(v[j])), static_cast<uint32_t>(__double2hiint(v[j]))};
        tm_st_x2(col + 2 * j, w);
    }
    tm_wait_st();
}
template <int RV>
__device__ __forceinline__ void tm_load_vec(uint32_t col, double (&v)[RV]) {
    uint32_t w[RV][2];
#pragma unroll
    for (int j = 0; j < RV; ++j) tm_ld_x2(col + 2 * j, w[j]);
    tm_wait_ld();
#pragma unroll
    for (int j = 0; j < RV; ++j) v[j] = __hiloint2double(static_cast<int>(w[j][1]), static_cast<int>(w[j][0]));
}

// Gather from the warp's X region: `xaddr` is its 32-bit shared address,
// aligned to a power of two above every offset, so the low step's address is
// one LOP3 ((w & 0x7FFF) | xaddr, which also drops the end flag) and the high
// step's one IMAD.HI ((w * 2^16) >> 32 + xaddr).
__device__ __forceinline__ uint32_t gaddr_lo(uint32_t w, uint32_t xaddr) { return (w & 0x7FFFu) | xaddr; }
__device__ __forceinline__ uint32_t gaddr_hi(uint32_t w, uint32_t xaddr) {
    uint32_t a;
    asm("mad.hi.u32 %0, %1, 65536, %2;" : "=r"(a) : "r"(w), "r"(xaddr));
    return a;
}
__device__ __forceinline__ double lds64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

// Everything a warp needs to run one SpMV of its group.
template <int RV>
struct TmemWarp {
    double* Xs;             // gather vector copies (+ trash slot), this warp (generic)
    double* Ys;             // row sums, lane-major, this warp
    uint32_t xaddr;         // shared address of Xs (aligned, see gaddr_lo)
    uint32_t xy[RV];        // copy-0 gather slot | Y slot << 16 of row slot j
    uint32_t x1[(RV + 1) / 2];  // copy-1 gather slots (CP = 2), row slots 2i | 2i+1 << 16
    uint32_t xyT[RV];       // BiCG pair: the same for p~ and the A^T outputs
    uint32_t x1T[(RV + 1) / 2];
    int lane;
    int ylane;              // this lane's column in the team's lane-major Y (32 * warp-in-team + lane)
    uint32_t wcol, vcol;    // TMEM addresses: words, this warp's values
    uint32_t dcol;          // BiCGSTAB: D^-1 (2*RV columns after the values)
    int S;
    int ystream;            // Y slots per row stream
};

// One 4-step chunk: words w0 (steps 0|1) and w1 (steps 2|3), values v[0..8);
// gathers issued first, then the ordered multiply-add chain(s).
//   ST = 1: one row at a time; rows end on step 1 (flag: bit 15 of w0) or 3
//           (bit 15 of w1).
//   ST = 2: two rows at a time, stream 0 on steps 0 and 2, stream 1 on steps 1
//           and 3 -- two independent DADD chains; stream 0 rows end on step 2
//           (flag in w0), stream 1 rows on step 3 (flag in w1).
template <int ST, int LW>
__device__ __forceinline__ void tmem_chunk4(uint32_t xaddr, uint32_t w0, uint32_t w1, const uint32_t* v,
                                            double (&acc)[ST], double* (&yp)[ST]) {
    const double x0 = lds64(gaddr_lo(w0, xaddr));
    const double x1 = lds64(gaddr_hi(w0, xaddr));
    const double x2 = lds64(gaddr_lo(w1, xaddr));
    const double x3 = lds64(gaddr_hi(w1, xaddr));
    const double a0 = __hiloint2double(static_cast<int>(v[1]), static_cast<int>(v[0]));
    const double a1 = __hiloint2double(static_cast<int>(v[3]), static_cast<int>(v[2]));
    const double a2 = __hiloint2double(static_cast<int>(v[5]), static_cast<int>(v[4]));
    const double a3 = __hiloint2double(static_cast<int>(v[7]), static_cast<int>(v[6]));
    if constexpr (ST == 1) {
        acc[0] = dadd(acc[0], dmul(a0, x0));
        acc[0] = dadd(acc[0], dmul(a1, x1));
        if (w0 & 0x8000u) {
            *yp[0] = acc[0];
            yp[0] += LW;
            acc[0] = 0.0;
        }
        acc[0] = dadd(acc[0], dmul(a2, x2));
        acc[0] = dadd(acc[0], dmul(a3, x3));
        if (w1 & 0x8000u) {
            *yp[0] = acc[0];
            yp[0] += LW;
            acc[0] = 0.0;
        }
    } else {
        acc[0] = dadd(acc[0], dmul(a0, x0));
        acc[1] = dadd(acc[1], dmul(a1, x1));
        acc[0] = dadd(acc[0], dmul(a2, x2));
        if (w0 & 0x8000u) {
            *yp[0] = acc[0];
            yp[0] += LW;
            acc[0] = 0.0;
        }
        acc[1] = dadd(acc[1], dmul(a3, x3));
        if (w1 & 0x8000u) {
            *yp[1] = acc[1];
            yp[1] += LW;
            acc[1] = 0.0;
        }
    }
}

// Publish x into every copy of the gather vector: copy-0 slot in the low half
// of xy[j], copy-1 slot in x1 (two row slots per word).
template <int CP, int RV>
__device__ __forceinline__ void tmem_publish(double* Xs, const uint32_t (&xy)[RV], const uint32_t (&x1)[(RV + 1) / 2],
                                             const double (&x)[RV]) {
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        Xs[xy[j] & 0xFFFFu] = x[j];
        if constexpr (CP == 2) Xs[(x1[j >> 1] >> (16 * (j & 1))) & 0xFFFFu] = x[j];
    }
}

// Walk the TMEM-resident schedule (8 steps per tcgen05.ld pair, then a 4-step
// tail; other warps hide the latency), row sums into Y.
template <int ST, int LW, int RV>
__device__ __forceinline__ void tmem_walk(const TmemWarp<RV>& tw) {
    double* yp[ST];
    double acc[ST];
#pragma unroll
    for (int s = 0; s < ST; ++s) {
        yp[s] = tw.Ys + s * tw.ystream + tw.ylane;
        acc[s] = 0.0;
    }
    int t0 = 0;
    // unrolled 4x (32 steps per loop iteration): B200, 100k cells, M156
    // BiCGSTAB 590k vs 574k cell-solves/s, BiCG 543k vs 506k, M312 275k vs
    // 258k; 2x: 589k / 530k / 267k; 8x: 568k / 536k / 256k
#pragma unroll 4
    for (; t0 + 8 <= tw.S; t0 += 8) {
        uint32_t w[4], v[16];
        tm_ld_x4(tw.wcol + (t0 >> 1), w);
        tm_ld_x16(tw.vcol + 2 * t0, v);
        tm_wait_ld();
        tmem_chunk4<ST, LW>(tw.xaddr, w[0], w[1], v, acc, yp);
        tmem_chunk4<ST, LW>(tw.xaddr, w[2], w[3], v + 8, acc, yp);
    }
    if (t0 < tw.S) {
        uint32_t w[2], v[8];
        tm_ld_x2(tw.wcol + (t0 >> 1), w);
        tm_ld_x8(tw.vcol + 2 * t0, v);
        tm_wait_ld();
        tmem_chunk4<ST, LW>(tw.xaddr, w[0], w[1], v, acc, yp);
    }
}

// y = A x (for a BiCG pair schedule the A^T stream runs on whatever p~ holds
// and its outputs are ignored).
template <int ST, int CP, int W, int RV>
__device__ __forceinline__ void tmem_spmv(const TmemWarp<RV>& tw, const Team<W>& tm, const double (&x)[RV],
                                          double (&y)[RV]) {
    tmem_publish<CP>(tw.Xs, tw.xy, tw.x1, x);
    tm.sync();
    tmem_walk<ST, 32 * W>(tw);
    tm.sync();
#pragma unroll
    for (int j = 0; j < RV; ++j) y[j] = tw.Ys[tw.xy[j] >> 16];
}

// BiCG's two products in one pass of the pair schedule: A p on stream 0,
// A^T p~ on stream 1 (bc_tmem_plan.cpp, pair mode).
template <int CP, int W, int RV>
__device__ __forceinline__ void tmem_spmv_pair(const TmemWarp<RV>& tw, const Team<W>& tm, const double (&pv)[RV],
                                               const double (&ps)[RV], double (&ap)[RV], double (&atps)[RV]) {
    tmem_publish<CP>(tw.Xs, tw.xy, tw.x1, pv);
    tmem_publish<CP>(tw.Xs, tw.xyT, tw.x1T, ps);
    tm.sync();
    tmem_walk<2, 32 * W>(tw);
    tm.sync();
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        ap[j] = tw.Ys[tw.xy[j] >> 16];
        atps[j] = tw.Ys[tw.xyT[j] >> 16];
    }
}

// Reduce NV values over the group: team_reduce<W = 1> with its
// validity selects dropped -- rows >= n already hold +0.0 by the zero
// invariant, exactly the value team_reduce substitutes -- and P = 32 * R >= 32
// known at compile time: lane tree over R slots, then the xor butterfly.
template <int NV, int R, int RV>
__device__ __forceinline__ void tmem_reduce(const double (&vals)[NV][RV], double (&out)[NV]) {
    static_assert(R >= 1 && RV <= R, "row slots beyond the tree");
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        double t[R];
#pragma unroll
        for (int j = 0; j < R; ++j) t[j] = j < RV ? vals[v][j < RV ? j : 0] : 0.0;
#pragma unroll
        for (int stride = R / 2; stride >= 1; stride /= 2)
#pragma unroll
            for (int j = 0; j < stride; ++j) t[j] = dadd(t[j], t[j + stride]);
        out[v] = t[0];
    }
#pragma unroll
    for (int mask = 16; mask >= 1; mask >>= 1)
#pragma unroll
        for (int v = 0; v < NV; ++v) out[v] = dadd(out[v], __shfl_xor_sync(0xffffffffu, out[v], mask));
}

// Two values through the xor butterfly with 6 instead of 10 64-bit shuffles:
// at mask 16 each lane sends the value its partner keeps -- lanes < 16 keep
// value 0, lanes >= 16 value 1 -- so masks 8..1 run one value per lane, and a
// last xor-16 shuffle hands every lane the other half's result.  Every dadd
// has the operands of tmem_reduce's butterfly (own value first, partner
// second; the xor butterfly leaves the same bits in every lane), so the
// results are bit-identical.  Measured neutral on the bench (586.3k both
// ways, B200): the kernel is not bound by its shuffles.  The chain is one
// shuffle longer, so the latency kernel keeps tmem_reduce.
template <int R, int RV>
__device__ __forceinline__ void tmem_reduce2(const double (&vals)[2][RV], double (&out)[2]) {
    static_assert(R >= 1 && RV <= R, "row slots beyond the tree");
    double o[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        double t[R];
#pragma unroll
        for (int j = 0; j < R; ++j) t[j] = j < RV ? vals[v][j < RV ? j : 0] : 0.0;
#pragma unroll
        for (int stride = R / 2; stride >= 1; stride /= 2)
#pragma unroll
            for (int j = 0; j < stride; ++j) t[j] = dadd(t[j], t[j + stride]);
        o[v] = t[0];
    }
    const bool upper = (threadIdx.x & 16u) != 0;
    double keep = upper ? o[1] : o[0];
    keep = dadd(keep, __shfl_xor_sync(0xffffffffu, upper ? o[0] : o[1], 16));
#pragma unroll
    for (int mask = 8; mask >= 1; mask >>= 1) keep = dadd(keep, __shfl_xor_sync(0xffffffffu, keep, mask));
    const double other = __shfl_xor_sync(0xffffffffu, keep, 16);
    out[0] = upper ? other : keep;
    out[1] = upper ? keep : other;
}

// W > 1: team_reduce (per-lane tree, one cross-warp step through shared
// memory, xor butterfly -- the same tree order for any team width).
template <int NV, int W, int R, int RV>
__device__ __forceinline__ void tmem_reduce(Ctx<W, R, RV>& c, const double (&vals)[NV][RV], double (&out)[NV]) {
    if constexpr (W == 1 && NV == 2)
        tmem_reduce2<R, RV>(vals, out);
    else if constexpr (W == 1)
        tmem_reduce<NV, R, RV>(vals, out);
    else
        team_reduce<NV>(c, vals, out);
}

template <int ST, int CP, int W, int R, int RV>
__device__ __forceinline__ double tmem_fresh_rms(Ctx<W, R, RV>& c, const TmemWarp<RV>& tw,
                                                 const double (&x)[RV], const double* bsrc) {
    double ax[RV];
    tmem_spmv<ST, CP>(tw, c.tm, x, ax);
    double sq[1][RV];
#pragma unroll
    for (int j = 0; j < RV; ++j) {
        const double bj = c.valid(j) ? bsrc[c.row(j)] : 0.0;
        const double ri = dsub(bj, ax[j]);
        sq[0][j] = dmul(ri, ri);
    }
    double out[1];
    tmem_reduce<1>(c, sq, out);
    return __dsqrt_rn(ddiv(out[0], static_cast<double>(c.n)));
}

template <int W, int R, int RV, int NT, int ST, int CP, int ALGO>
__global__ void __launch_bounds__(NT, 1) block_cells_tmem_kernel(const TmemParams p) {
    constexpr int LW = 32 * W;  // lanes per group (a team of W warps per cell)
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_taddr;
    __shared__ int s_group[16];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int quarter = warp % 4, slot = warp / 4;
    const int team = warp / W, wr = warp % W;  // team = consecutive warps: quarter % W == wr
    int32_t* s_vidx = reinterpret_cast<int32_t*>(smem);  // S*LW
    // X regions (one per team, each aligned to xalign), then Y regions, then
    // (W > 1) the cross-warp reduction buffers
    const uint32_t s_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const uint32_t x_area = (s_base + sizeof(int32_t) * p.S * LW + p.xalign - 1) &
                            ~static_cast<uint32_t>(p.xalign - 1);
    const int nteams = blockDim.x / LW;
    double* s_y = reinterpret_cast<double*>(smem + (x_area - s_base) + static_cast<size_t>(nteams) * p.xalign);
    double* s_red = s_y + static_cast<size_t>(nteams) * p.yslots;

    for (int i = threadIdx.x; i < p.S * LW; i += blockDim.x) s_vidx[i] = p.vidx[i];
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
    TmemWarp<RV> tw;
    tw.wcol = lane_base;  // words: columns [0, S/2)
    // per warp: 2S value columns (+ 2*RV for BiCGSTAB's D^-1)
    const uint32_t warp_cols = 2u * p.S + (ALGO == kBiCGStab ? 2u * RV : 0u);
    tw.vcol = lane_base + p.S / 2 + warp_cols * static_cast<uint32_t>(slot);
    tw.dcol = tw.vcol + 2u * p.S;
    if (slot == 0) {  // words of this quarter's team role into TMEM once (same for every group)
        const uint16_t* wsrc = p.words + wr * 32 + lane;
        for (int t0 = 0; t0 < p.S; t0 += 4) {
            uint32_t w[2];
            w[0] = wsrc[t0 * LW] | (static_cast<uint32_t>(wsrc[(t0 + 1) * LW]) << 16);
            w[1] = wsrc[(t0 + 2) * LW] | (static_cast<uint32_t>(wsrc[(t0 + 3) * LW]) << 16);
            tm_st_x2(tw.wcol + (t0 >> 1), w);
        }
        tm_wait_st();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    const bool active = slot < p.cells_per_quarter;
    Ctx<W, R, RV> c;
    c.tm.id = team;
    c.tm.w = wr;
    c.tm.lane = lane;
    c.tm.tid = wr * 32 + lane;
    c.n = p.n;
    c.P = p.P;
    c.red = s_red + static_cast<size_t>(team) * (2 * 4 * LW);
    c.red_buf = 0;
    tw.xaddr = x_area + static_cast<uint32_t>(team * p.xalign);
    tw.Xs = reinterpret_cast<double*>(smem + (tw.xaddr - s_base));
    tw.Ys = s_y + static_cast<size_t>(team) * p.yslots;
    tw.lane = lane;
    tw.ylane = wr * 32 + lane;
    tw.S = p.S;
    tw.ystream = p.ystream;
#pragma unroll
    for (int j = 0; j < RV; ++j) tw.xy[j] = p.lane_xy[c.row(j)];
#pragma unroll
    for (int i = 0; i < (RV + 1) / 2; ++i) tw.x1[i] = CP == 2 ? p.lane_x1[(i * W + wr) * 32 + lane] : 0u;
#pragma unroll
    for (int j = 0; j < RV; ++j) tw.xyT[j] = ALGO == kBiCG ? p.lane_xyT[c.row(j)] : 0u;
#pragma unroll
    for (int i = 0; i < (RV + 1) / 2; ++i)
        tw.x1T[i] = (ALGO == kBiCG && CP == 2) ? p.lane_x1T[(i * W + wr) * 32 + lane] : 0u;
    for (int i = c.tm.tid; i < p.xslots; i += LW) tw.Xs[i] = 0.0;  // zero slots stay +0.0
    for (int i = c.tm.tid; i < p.yslots; i += LW) tw.Ys[i] = 0.0;
    if (active) c.tm.sync();
    const double smax = p.sigma_max;

    while (active) {
        int gl;
        if constexpr (W == 1) {
            unsigned int gv = 0;
            if (lane == 0) gv = atomicAdd(p.counter, 1u);
            gl = static_cast<int>(__shfl_sync(0xffffffffu, gv, 0));
        } else {
            if (c.tm.tid == 0) s_group[team] = static_cast<int>(atomicAdd(p.counter, 1u));
            c.tm.sync();
            gl = s_group[team];
            c.tm.sync();
        }
        if (gl >= p.group_count) break;
        if (p.gate.ready) {
            if (c.tm.tid == 0) gate_wait(p.gate, gl);
            c.tm.sync();
        }
        const int64_t cell0 = p.cell_offset + static_cast<int64_t>(gl) * p.kc;
        const double* src = p.values + cell0 * p.nnz;
        const double* bsrc = p.rhs + cell0 * p.species;

        // stage this group's values into TMEM in schedule order (once per solve)
        for (int t0 = 0; t0 < p.S; t0 += 4) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int vi = s_vidx[(t0 + u) * LW + c.tm.tid];
                const double a = vi >= 0 ? __ldg(src + vi) : 0.0;
                v[2 * u] = static_cast<uint32_t>(__double2loint(a));
                v[2 * u + 1] = static_cast<uint32_t>(__double2hiint(a));
            }
            tm_st_x8(tw.vcol + 2 * t0, v);
        }
        tm_wait_st();
        __syncwarp();

        double x[RV];
#pragma unroll
        for (int j = 0; j < RV; ++j) x[j] = 0.0;
        int iters = 0;
        bool conv = false, brk = false;
        double fres = 0.0;
        if constexpr (ALGO == kBiCGStab) {
            {  // D^-1 into TMEM (read back where used: frees 2*RV registers)
                double dinv[RV];
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    const int di = c.valid(j) ? p.didx[c.row(j)] : -1;
                    const double d = di >= 0 ? __ldg(src + di) : 0.0;
                    dinv[j] = c.valid(j) ? (d != 0.0 ? ddiv(1.0, d) : 1.0) : 0.0;
                }
                tm_store_vec(tw.dcol, dinv);
            }
            double r[RV], rh[RV], pv[RV], v[RV];
            {
                double ax[RV];
                tmem_spmv<ST, CP>(tw, c.tm, x, ax);
    #pragma unroll
                for (int j = 0; j < RV; ++j) {
                    const double bj = c.valid(j) ? __ldcs(bsrc + c.row(j)) : 0.0;
                    r[j] = dadd(bj, -ax[j]);  // 1*b + (-1)*Ax; rows >= n: 0 + -0 = +0
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
                tmem_reduce<2>(c, q, o);
                sigma = o[0];
                rho_next = o[1];
            }
            if (sigma <= smax) {
                fres = tmem_fresh_rms<ST, CP>(c, tw, x, bsrc);
                conv = fres <= p.tol;
            }
            if (!conv) {
                double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
                double aw = ddiv(alpha, omega);  // alpha/omega of beta, computed as soon as omega is known
                for (int it = 1; it <= p.max_iter; ++it) {
                    const double rho = rho_next;
                    if (scalar_breaks(rho)) { brk = true; break; }
                    const double beta = dmul(ddiv(rho, rho_prev), aw);
                    double y[RV], dinv[RV];
                    tm_load_vec(tw.dcol, dinv);
    #pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        pv[j] = dadd(r[j], dmul(beta, dsub(pv[j], dmul(omega, v[j]))));
                        y[j] = dmul(dinv[j], pv[j]);
                    }
                    tmem_spmv<ST, CP>(tw, c.tm, y, v);
                    double den;
                    {
                        double q[1][RV], o[1];
    #pragma unroll
                        for (int j = 0; j < RV; ++j) q[0][j] = dmul(rh[j], v[j]);
                        tmem_reduce<1>(c, q, o);
                        den = o[0];
                    }
                    if (scalar_breaks(den)) { brk = true; break; }
                    alpha = ddiv(rho, den);
                    double z[RV], dinv2[RV];
                    tm_load_vec(tw.dcol, dinv2);
    #pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        r[j] = dsub(r[j], dmul(alpha, v[j]));                  // r now holds s
                        z[j] = dmul(dinv2[j], r[j]);
                        x[j] = dadd(x[j], dmul(alpha, dmul(dinv2[j], pv[j])));  // y = dinv*p recomputed
                    }
                    double t[RV];
                    tmem_spmv<ST, CP>(tw, c.tm, z, t);
                    double tt, ts;
                    {
                        double q[2][RV], o[2];
    #pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(t[j], t[j]);
                            q[1][j] = dmul(t[j], r[j]);
                        }
                        tmem_reduce<2>(c, q, o);
                        tt = o[0];
                        ts = o[1];
                    }
                    if (tt != 0.0 && scalar_breaks(tt)) { brk = true; break; }
                    omega = tt == 0.0 ? 0.0 : ddiv(ts, tt);
                    aw = ddiv(alpha, omega);  // next beta's factor, off the critical path
                    double dinv3[RV];
                    tm_load_vec(tw.dcol, dinv3);
    #pragma unroll
                    for (int j = 0; j < RV; ++j) {
                        x[j] = dadd(x[j], dmul(omega, dmul(dinv3[j], r[j])));  // z = dinv*s recomputed
                        r[j] = dsub(r[j], dmul(omega, t[j]));
                    }
                    rho_prev = rho;
                    iters = it;
                    {
                        double q[2][RV], o[2];
    #pragma unroll
                        for (int j = 0; j < RV; ++j) {
                            q[0][j] = dmul(r[j], r[j]);
                            q[1][j] = dmul(rh[j], r[j]);
                        }
                        tmem_reduce<2>(c, q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (sigma <= smax) {
                        const double f = tmem_fresh_rms<ST, CP>(c, tw, x, bsrc);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                    if (scalar_breaks(omega)) { brk = true; break; }
                }
                if (!conv) {
                    fres = tmem_fresh_rms<ST, CP>(c, tw, x, bsrc);
                    conv = !brk && fres <= p.tol;
                }
            }
        } else {
            // BiCG, bicg.cpp:42-142 operation for operation (as block_cells_kernel's
            // kBiCG branch), A p and A^T p~ in one pass of the pair schedule
            double r[RV], rs[RV], pv[RV], ps[RV];
            {
                double ax[RV];
                tmem_spmv<ST, CP>(tw, c.tm, x, ax);
#pragma unroll
                for (int j = 0; j < RV; ++j) {
                    const double bj = c.valid(j) ? __ldcs(bsrc + c.row(j)) : 0.0;
                    r[j] = dadd(bj, -ax[j]);  // 1*b + (-1)*Ax; rows >= n: 0 + -0 = +0
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
                tmem_reduce<2>(c, q, o);
                sigma = o[0];
                rho_next = o[1];
            }
            if (sigma <= smax) {
                fres = tmem_fresh_rms<ST, CP>(c, tw, x, bsrc);
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
                    tmem_spmv_pair<CP>(tw, c.tm, pv, ps, ap, atps);
                    double den;
                    {
                        double q[1][RV], o[1];
#pragma unroll
                        for (int j = 0; j < RV; ++j) q[0][j] = dmul(ps[j], ap[j]);
                        tmem_reduce<1>(c, q, o);
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
                        tmem_reduce<2>(c, q, o);
                        sigma = o[0];
                        rho_next = o[1];
                    }
                    if (!isfinite(sigma)) { brk = true; break; }
                    if (sigma <= smax) {
                        const double f = tmem_fresh_rms<ST, CP>(c, tw, x, bsrc);
                        if (f <= p.tol) {
                            fres = f;
                            conv = true;
                            break;
                        }
                    }
                }
                if (!conv) {
                    fres = tmem_fresh_rms<ST, CP>(c, tw, x, bsrc);
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
            p.g_iters[g] = iters;
            p.g_rms[g] = fres;
            p.g_flags[g] = static_cast<uint8_t>((conv ? 1 : 0) | (brk ? 2 : 0));
        }
        c.tm.sync();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "r"(512));
}

}  // namespace bc
