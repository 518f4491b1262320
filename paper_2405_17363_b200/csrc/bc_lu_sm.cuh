// bc_lu_sm.cuh -- breakdown fallback for groups made of s x s blocks that fit
// in shared memory (block-diagonal Block-cells(k) groups and one-cell groups
// at CB05 size: 156 x 157 doubles = 196 KB), in two kernels.
//
// bc_lu.cuh's lu_fallback_kernel keeps each block in global scratch and runs
// factorization, forward and backward substitution in one CTA of 256 threads
// (three per SM).  Profiled on Block-cells(N) M156 (ncu, 10k cells): ~840k
// warp instructions and ~1.7M cycles per 156 x 156 block, 60% of scheduler
// cycles with no eligible warp -- every phase waits on L2 round trips and
// barriers, and the backward substitution (a 12k-step ordered DSUB chain per
// block, ~60 us) holds the CTA while one lane per block works.  Here:
//
//   lu_sm_factor_kernel (512 threads, one CTA per SM): per group, block by
//     block, densify into shared memory, factor there (panels of 16 columns,
//     thread-per-row panel updates, U12 by thread-per-column triangular solves,
//     A22 in 4 x 4 register micro-tiles), forward-substitute, and park the
//     factors in scratch and the forward result in x_out;
//   lu_sm_solve_kernel (one warp per block, many CTAs per SM): the backward
//     chains of all blocks at once, the exact redo of a block whose -0 row sum
//     a later negative x flips, the non-finite check and the residual.
//
// Arithmetic is bc_lu.cuh's, operation for operation: every element receives
// a_ij -= l_ik u_kj one k at a time in ascending k, each product and
// difference rounded separately, pivots by largest magnitude with ties to the
// lowest row (dense_lu.cpp:18-63), the same sign-of-zero replay between blocks
// and the same status protocol (1 singular, 2 non-finite -> dense rerun).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bc_lu.cuh"

namespace bc {

#ifdef BC_LU_PROFILE
// phase cycles of CTA 0 (thread 0's clock), tools/luprof.cu
__device__ unsigned long long bc_lu_prof[64];
#define LU_MARK(i)                                         \
    do {                                                   \
        if (blockIdx.x == 0 && threadIdx.x == 0) {         \
            const long long now_ = clock64();              \
            bc_lu_prof[i] += static_cast<unsigned long long>(now_ - lu_t0_); \
            lu_t0_ = now_;                                 \
        }                                                  \
    } while (0)
#define LU_PROF_START long long lu_t0_ = clock64()
#define LU_TICKS_DECL long long lu_tk_[4] = {0, 0, 0, 0}, lu_tq_ = clock64()
#define LU_TICK(i)                           \
    do {                                     \
        const long long now_ = clock64();    \
        lu_tk_[i] += now_ - lu_tq_;          \
        lu_tq_ = now_;                       \
    } while (0)
#define LU_TICKS_FLUSH                                                              \
    do {                                                                            \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                             \
            for (int q_ = 0; q_ < 4; ++q_) bc_lu_prof[16 + 4 * (threadIdx.x >> 5) + q_] += lu_tk_[q_]; \
    } while (0)
#else
#define LU_TICKS_DECL
#define LU_TICK(i) \
    do {           \
    } while (0)
#define LU_TICKS_FLUSH \
    do {               \
    } while (0)
#define LU_MARK(i) \
    do {           \
    } while (0)
#define LU_PROF_START
#endif

constexpr int kLuSmThreads = 256;
constexpr int kLuSmPanel = 16;
constexpr int kLuSmMaxRows = 160;                     // blocks up to 160 x 160 (196 KB at 156)
constexpr int kLuSmColsPerLane = kLuSmMaxRows / 32;  // A22: a lane's 32-strided columns

// leading dimension of a block in shared memory: odd, so a column walk (one
// row per thread) touches distinct banks
__host__ __device__ constexpr int lu_sm_ld(int s) { return s | 1; }

// A22 -= L21 U12 over the panel [k0, k1): row bands of 4, one warp per band,
// lane L holding columns k1 + L + 32q (q < NQ); per element the panel's
// updates one k at a time in ascending order.  Rows past the edge read the
// zero padding rows and are never stored.
template <int NQ>
__device__ __forceinline__ void lu_sm_a22(double* a, const int n, const int ld, const int k0, const int k1) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int m = n - k1, bands = (m + 3) >> 2, j0 = k1 + lane;
    bool cok[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) cok[q] = j0 + 32 * q < n;
    for (int band = warp; band < bands; band += nw) {
        const int i0 = k1 + 4 * band;
        double acc[4][NQ];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[r][q] = cok[q] ? a[(i0 + r) * ld + j0 + 32 * q] : 0.0;
#pragma unroll 4
        for (int kk = k0; kk < k1; ++kk) {
            double l[4], u[NQ];
#pragma unroll
            for (int r = 0; r < 4; ++r) l[r] = a[(i0 + r) * ld + kk];
#pragma unroll
            for (int q = 0; q < NQ; ++q) u[q] = cok[q] ? a[kk * ld + j0 + 32 * q] : 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < NQ; ++q) acc[r][q] = __dsub_rn(acc[r][q], __dmul_rn(l[r], u[q]));
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (i0 + r < n && cok[q]) a[(i0 + r) * ld + j0 + 32 * q] = acc[r][q];
    }
}

// a / b as __ddiv_rn for b != 0, with a zero dividend answered directly:
// __ddiv_rn sends a zero quotient down its slow path (~1,000 cycles), and most
// entries below a sparse block's diagonal are zero.  0 / b (b finite or
// infinite, nonzero) is a zero with the sign sign(a) ^ sign(b); 0 / NaN is
// left to __ddiv_rn.
__device__ __forceinline__ double lu_div(const double a, const double b) {
    if (a == 0.0 && !isnan(b))
        return __longlong_as_double((__double_as_longlong(a) ^ __double_as_longlong(b)) &
                                    static_cast<long long>(0x8000000000000000ull));
    return __ddiv_rn(a, b);
}

// Named barrier over the first `count` threads (the row owners).
__device__ __forceinline__ void lu_sm_bar(int count) { asm volatile("bar.sync 1, %0;" ::"r"(count) : "memory"); }

// Factor the n x n block `a` (shared, leading dimension ld, at least 4 rows of
// readable padding after it) in place; perm[] (shared) starts as the identity
// and records the row swaps.  Returns false (uniformly) when the block is
// exactly singular (dense_lu.cpp:35).  Per panel of 16 columns:
//   * the row owners (thread i holds row i: the first ceil(n/32) warps, synced
//     by a named barrier) factor the panel: each owner's |a_ik| joins its
//     warp's argmax butterfly, the warps' winners meet in shared memory, the
//     panel parts of rows k and piv swap, and every owner below k forms
//     l = a_ik / pivot and its row's panel update with the pivot row's
//     entries in registers -- then the next column's candidate at once;
//   * all threads: the panel's row swaps, in order, on the other columns;
//     U12 by thread-per-column triangular solves; A22 by row bands of 4, one
//     warp per band, each lane a 4 x ceil(m/32) micro-tile of 32-strided
//     columns (conflict-free loads of the pivot rows, broadcast L loads).
__device__ bool lu_sm_factor(double* a, const int n, const int ld, int* perm, int* s_piv, int* s_flag,
                             int* posof, double* magk, double* prow_s) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    // every warp owns a contiguous run of rows (lanes [0, per)): the panel's
    // work spreads evenly over the four SM sub-partitions
    const int nwarps = nt >> 5, per = (n + nwarps - 1) / nwarps;
    LU_PROF_START;
    for (int k0 = 0; k0 < n; k0 += kLuSmPanel) {
        const int k1 = min(n, k0 + kLuSmPanel), K = k1 - k0;
        // ---- panel: columns [k0, k1), rows [k0, n).  Every thread owns at most one
        // row and keeps the row's panel part in registers for the whole panel;
        // rows stay where they are (each owner tracks its row's position, the
        // reference's swapped order, which breaks magnitude ties).  Per column:
        // barrier A; every warp scans the published (magnitude, position) pairs
        // the same way (uniform pivot); the pivot row's owner publishes its
        // panel part; barrier B; the owners below form l = a_ik / pivot, update
        // their registers and publish their next candidate.
        {
            const bool owner = lane < per && warp * per + lane < n;
            const int i = owner ? warp * per + lane : n;  // physical row (n: none)
            int pos = i;                                  // its position
            double v[kLuSmPanel];
#pragma unroll
            for (int jj = 0; jj < kLuSmPanel; ++jj) v[jj] = (owner && jj < K) ? a[i * ld + k0 + jj] : 0.0;
            if (owner) {
                posof[i] = pos;
                magk[i] = fabs(v[0]);
            }
            if (tid == 0) *s_flag = 0;  // read after barrier B at the earliest
            LU_TICKS_DECL;
#pragma unroll
            for (int kk = 0; kk < kLuSmPanel; ++kk) {
                if (kk >= K) break;  // uniform
                const int k = k0 + kk, cur = kk & 1;
                __syncthreads();  // A: the candidates of column k are published
                LU_TICK(0);
                // a warp whose rows are all pivoted has nothing left in this panel
                // but the barriers (uniform per warp)
                if (!__any_sync(0xffffffffu, i < n && pos >= k)) {
                    __syncthreads();  // B
                    if (*s_flag) break;  // singular (uniform)
                    if (kk + 1 < K && i < n) posof[(cur ^ 1) * kLuSmMaxRows + i] = pos;  // (< k: never a candidate)
                    continue;
                }
                // the scan: largest magnitude, ties to the lowest position, NaN
                // skipped; the row at position k and whether it holds a NaN there
                int pr_[kLuSmMaxRows / 32];
                double mg_[kLuSmMaxRows / 32];
#pragma unroll
                for (int q = 0; q < kLuSmMaxRows / 32; ++q) {
                    pr_[q] = posof[cur * kLuSmMaxRows + lane + 32 * q];
                    mg_[q] = magk[cur * kLuSmMaxRows + lane + 32 * q];
                }
                double bm = -1.0;
                unsigned bp = 0x7fffffffu;
                int brow = 0, krow = -1;
                bool nan_k = false;
#pragma unroll
                for (int q = 0; q < kLuSmMaxRows / 32; ++q) {
                    const int r = lane + 32 * q;
                    const bool live = r < n;
                    const bool isk = live && pr_[q] == k;
                    krow = isk ? r : krow;
                    nan_k = nan_k || (isk && isnan(mg_[q]));
                    const bool better = live && pr_[q] >= k &&
                                        (mg_[q] > bm || (mg_[q] == bm && static_cast<unsigned>(pr_[q]) < bp));
                    bm = better ? mg_[q] : bm;
                    bp = better ? static_cast<unsigned>(pr_[q]) : bp;
                    brow = better ? r : brow;
                }
                // (hi, lo) word order = magnitude order for non-negative doubles;
                // hi | 1 << 31 keeps 0 for "none"
                const unsigned bh = bm >= 0.0 ? (static_cast<unsigned>(__double2hiint(bm)) | 0x80000000u) : 0u;
                const unsigned bl = bm >= 0.0 ? static_cast<unsigned>(__double2loint(bm)) : 0u;
                const unsigned H = __reduce_max_sync(0xffffffffu, bh);
                const unsigned L = __reduce_max_sync(0xffffffffu, bh == H ? bl : 0u);
                const unsigned P = __reduce_min_sync(0xffffffffu, (bh == H && bl == L) ? bp : 0x7fffffffu);
                const unsigned wb = __ballot_sync(0xffffffffu, bh == H && bl == L && bp == P);
                const unsigned kb = __ballot_sync(0xffffffffu, krow >= 0);
                const bool nan_any = __any_sync(0xffffffffu, nan_k);
                // dense_lu.cpp:32-41: largest magnitude in column k, ties to the
                // lowest position; a NaN at (k, k) fails every comparison: pivot k
                int pp = k, pr = __shfl_sync(0xffffffffu, krow, __ffs(kb) - 1);
                if (!nan_any) {
                    if (H == 0x80000000u && L == 0u) {  // the largest magnitude is 0: dense_lu.cpp:35
                        if (lane == 0) *s_flag = 1;
                        __syncthreads();  // B: every thread then leaves (below)
                        break;
                    }
                    pp = static_cast<int>(P);
                    pr = __shfl_sync(0xffffffffu, brow, __ffs(wb) - 1);
                }
                LU_TICK(1);
                if (i == pr) {  // the pivot row's panel part, for everyone
                    s_piv[kk] = pp;
#pragma unroll
                    for (int jj = kk; jj < kLuSmPanel; ++jj) prow_s[cur * kLuSmPanel + jj] = v[jj];
                }
                if (pos == pp) pos = k;
                else if (pos == k) pos = pp;
                __syncthreads();  // B: the pivot row is published
                if (i < n && pos > k) {  // rows not yet pivoted: l = a_ik / pivot, the panel's rest
                    double u[kLuSmPanel];
#pragma unroll
                    for (int jj = kk; jj < kLuSmPanel; ++jj) u[jj] = prow_s[cur * kLuSmPanel + jj];
                    const double lk = lu_div(v[kk], u[kk]);
                    v[kk] = lk;
#pragma unroll
                    for (int jj = kk + 1; jj < kLuSmPanel; ++jj)
                        if (jj < K) v[jj] = __dsub_rn(v[jj], __dmul_rn(lk, u[jj]));
                }
                if (kk + 1 < K && i < n) {  // the next column's candidate (buffer cur ^ 1)
                    posof[(cur ^ 1) * kLuSmMaxRows + i] = pos;
                    magk[(cur ^ 1) * kLuSmMaxRows + i] = fabs(v[kk + 1 < kLuSmPanel ? kk + 1 : kk]);
                }
                LU_TICK(2);
            }
            LU_TICKS_FLUSH;
            if (owner) {
#pragma unroll
                for (int jj = 0; jj < kLuSmPanel; ++jj)
                    if (jj < K) a[i * ld + k0 + jj] = v[jj];
            }
        }
        __syncthreads();
        LU_MARK(0);
        if (*s_flag) return false;
        // ---- the panel's row swaps, in order, on every column (the panel's too:
        // its rows stayed in place), and on perm
        if (tid == nt - 1)
            for (int kk = 0; kk < K; ++kk) {
                const int pr = s_piv[kk];
                const int t = perm[k0 + kk];
                perm[k0 + kk] = perm[pr];
                perm[pr] = t;
            }
        for (int c = tid; c < n; c += nt) {
            for (int kk = 0; kk < K; ++kk) {
                const int pr = s_piv[kk];
                if (pr != k0 + kk) {
                    const double t = a[(k0 + kk) * ld + c];
                    a[(k0 + kk) * ld + c] = a[pr * ld + c];
                    a[pr * ld + c] = t;
                }
            }
        }
        __syncthreads();
        LU_MARK(1);
        if (k1 == n) break;
        // ---- U12: rows [k0, k1), columns [k1, n): a_ij -= l_ik u_kj for k = k0 .. i-1
        for (int j = k1 + tid; j < n; j += nt) {
            double u[kLuSmPanel];
#pragma unroll
            for (int i = 0; i < kLuSmPanel; ++i) u[i] = i < K ? a[(k0 + i) * ld + j] : 0.0;
#pragma unroll
            for (int kk = 0; kk < kLuSmPanel; ++kk)
#pragma unroll
                for (int i = kk + 1; i < kLuSmPanel; ++i)
                    if (i < K) u[i] = __dsub_rn(u[i], __dmul_rn(a[(k0 + i) * ld + k0 + kk], u[kk]));
#pragma unroll
            for (int i = 1; i < kLuSmPanel; ++i)
                if (i < K) a[(k0 + i) * ld + j] = u[i];
        }
        __syncthreads();
        LU_MARK(2);
        // ---- A22: rows and columns [k1, n); row bands of 4, one warp per band,
        // lane L holding columns k1 + L + 32q (q < ceil(m / 32))
        switch ((n - k1 + 31) >> 5) {
            case 1: lu_sm_a22<1>(a, n, ld, k0, k1); break;
            case 2: lu_sm_a22<2>(a, n, ld, k0, k1); break;
            case 3: lu_sm_a22<3>(a, n, ld, k0, k1); break;
            case 4: lu_sm_a22<4>(a, n, ld, k0, k1); break;
            default: lu_sm_a22<kLuSmColsPerLane>(a, n, ld, k0, k1); break;
        }
        __syncthreads();
        LU_MARK(3);
    }
    return true;
}

// Forward substitution L y = P b (dense_lu.cpp:53-57) on y[] (shared, holding
// P b), L in shared memory: row i subtracts j = 0..i-1 in order.
__device__ void lu_sm_forward(const double* a, const int n, const int ld, double* y) {
    const int i = threadIdx.x;
    for (int j = 0; j < n; ++j) {
        __syncthreads();
        if (i > j && i < n) y[i] = __dsub_rn(y[i], __dmul_rn(a[i * ld + j], y[j]));
    }
    __syncthreads();
}

// Dynamic shared memory of lu_sm_factor_kernel for s-row blocks.
__host__ __device__ constexpr size_t lu_sm_factor_smem(int s) {
    return sizeof(double) * (static_cast<size_t>(s + 4) * lu_sm_ld(s) + s) + sizeof(int) * ((s + 1) & ~1);
}

// Per group: blocks c = 0 .. kc-1 in order (the sign-of-zero replay of
// bc_lu.cuh flows from earlier blocks to later ones).  Status 1 = singular,
// 2 = non-finite (the host reruns the group densely), -1 = factored (the solve
// kernel finishes it).
__global__ void __launch_bounds__(kLuSmThreads, 1) lu_sm_factor_kernel(const LuParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_piv[kLuSmPanel], s_flag;
    __shared__ int posof[2 * kLuSmMaxRows];
    __shared__ double prow_s[2 * kLuSmPanel];
    __shared__ double magk[2 * kLuSmMaxRows];
    const LuEntry ent = p.entries[blockIdx.x];
    const int s = p.species, ld = lu_sm_ld(s), tid = threadIdx.x, nt = blockDim.x;
    double* a = reinterpret_cast<double*>(smem_raw);
    double* y = a + static_cast<size_t>(s + 4) * ld;  // 4 padding rows: A22's edge tiles read them
    int* perm = reinterpret_cast<int*>(y + s);
    double* lu = p.scratch + static_cast<size_t>(blockIdx.x) * p.stride;
    const double* vals = p.values + ent.cell0 * p.nnz;
    const double* b = p.rhs + ent.cell0 * s;
    double* yout = p.x_out + ent.cell0 * s;

    int bad = 0;  // finite inputs only (0 * inf would spread NaN across blocks)
    for (int64_t q = tid; q < static_cast<int64_t>(ent.kc) * p.nnz; q += nt) bad |= !isfinite(vals[q]);
    for (int q = tid; q < ent.kc * s; q += nt) bad |= !isfinite(b[q]);
    if (__syncthreads_or(bad)) {
        if (tid == 0) p.status[blockIdx.x] = 2;
        return;
    }
    bool neg_pivot = false, fwd_flip = false;
    LU_PROF_START;
    for (int c = 0; c < ent.kc; ++c) {
        // dense_lu.cpp:8-16 on this block (the off-diagonal blocks are zero)
        for (int q = tid; q < (s + 4) * ld; q += nt) a[q] = 0.0;
        for (int i = tid; i < s; i += nt) perm[i] = i;
        __syncthreads();
        const double* cv = vals + static_cast<int64_t>(c) * p.nnz;
        for (int i = tid; i < s; i += nt)
            for (int e = p.row_ptr[i]; e < p.row_ptr[i + 1]; ++e) {
                double v = cv[e];
                if (neg_pivot && is_neg_zero(v)) v = 0.0;  // an earlier block's negative pivot
                a[i * ld + p.col_idx[e]] = v;
            }
        __syncthreads();
        LU_MARK(4);
        if (!lu_sm_factor(a, s, ld, perm, s_piv, &s_flag, posof, magk, prow_s)) {
            if (tid == 0) p.status[blockIdx.x] = 1;
            return;
        }
        LU_MARK(5);
        int neg = 0, nonfinite = 0;
        for (int i = tid; i < s; i += nt) {
            const double* row = a + i * ld;
            for (int j = 0; j < s; ++j) nonfinite |= !isfinite(row[j]);
            neg |= signbit(row[i]) ? 1 : 0;
        }
        neg_pivot = __syncthreads_or(neg) || neg_pivot;
        if (__syncthreads_or(nonfinite)) {
            if (tid == 0) p.status[blockIdx.x] = 2;
            return;
        }
        for (int i = tid; i < s; i += nt) {
            double v = b[c * s + perm[i]];
            if (fwd_flip && is_neg_zero(v)) v = 0.0;
            y[i] = v;
        }
        LU_MARK(6);
        lu_sm_forward(a, s, ld, y);
        LU_MARK(7);
        int flip = 0;
        for (int i = tid; i < s; i += nt) {
            flip |= (signbit(a[i * ld + i]) != signbit(y[i])) ? 1 : 0;
            yout[c * s + i] = y[i];
        }
        fwd_flip = __syncthreads_or(flip) || fwd_flip;
        // park the factors for the solve kernel (row-major, leading dimension s)
        double* g = lu + static_cast<int64_t>(c) * s * s;
        for (int q = tid; q < s * s; q += nt) g[q] = a[(q / s) * ld + q % s];
        __syncthreads();
        LU_MARK(8);
    }
    if (tid == 0) p.status[blockIdx.x] = -1;
}

// Dynamic shared memory of lu_sm_solve_kernel: sum (n) | ycopy (n) | slots
// (max(padded n, warps x s)).
__host__ constexpr size_t lu_sm_solve_smem(int64_t n, int64_t pn, int warps, int s) {
    return sizeof(double) * (2 * n + (pn > static_cast<int64_t>(warps) * s ? pn : static_cast<int64_t>(warps) * s));
}

// One CTA of min(kc, 32) warps per factored group: the backward substitutions
// of all blocks at once, each assuming no later block has a negative x; then,
// last block first as in the reference, the rare block that summed a row to -0
// while a later x is negative is redone from its forward result; non-finite
// results go to the dense rerun; then the residual.
__global__ void __launch_bounds__(1024, 1) lu_sm_solve_kernel(const LuParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned s_zmask[64];
    if (p.status[blockIdx.x] != -1) return;  // singular or non-finite: nothing to finish (uniform)
    const LuEntry ent = p.entries[blockIdx.x];
    const int s = p.species, n = ent.kc * s, tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid / 32, nw = nt / 32;
    double* sum = reinterpret_cast<double*>(smem_raw);
    double* ycopy = sum + n;
    double* slots = ycopy + n;
    const double* lu = p.scratch + static_cast<size_t>(blockIdx.x) * p.stride;
    const double* vals = p.values + ent.cell0 * p.nnz;
    const double* b = p.rhs + ent.cell0 * s;
    double* xo = p.x_out + ent.cell0 * s;

    for (int i = tid; i < 64; i += nt) s_zmask[i] = 0u;
    for (int i = tid; i < n; i += nt) ycopy[i] = sum[i] = xo[i];
    __syncthreads();
    for (int c = warp; c < ent.kc; c += nw) {
        const bool z = lu_backward_warp(lu + static_cast<int64_t>(c) * s * s, s, sum + c * s, slots + warp * s, false);
        if (z && (tid % 32) == 0) atomicOr(&s_zmask[c / 32], 1u << (c % 32));
    }
    __syncthreads();
    if (tid < 32) {
        bool later_neg = false;
        for (int c = ent.kc - 1; c >= 0; --c) {
            double* xc = sum + c * s;
            if (later_neg && (s_zmask[c / 32] >> (c % 32) & 1u)) {
                for (int i = tid; i < s; i += 32) xc[i] = ycopy[c * s + i];
                __syncwarp();
                lu_backward_warp(lu + static_cast<int64_t>(c) * s * s, s, xc, slots, true);
            }
            int neg = 0;
            for (int i = tid; i < s; i += 32) neg |= signbit(xc[i]) ? 1 : 0;
            later_neg = __any_sync(0xffffffffu, neg) || later_neg;
        }
    }
    __syncthreads();
    int nonfinite = 0;
    for (int i = tid; i < n; i += nt) nonfinite |= !isfinite(sum[i]);
    if (__syncthreads_or(nonfinite)) {
        if (tid == 0) p.status[blockIdx.x] = 2;
        return;
    }
    for (int i = tid; i < n; i += nt) xo[i] = sum[i];
    lu_group_residual(p, ent, n, vals, b, sum, slots);
}

}  // namespace bc
