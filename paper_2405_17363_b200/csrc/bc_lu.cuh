// bc_lu.cuh -- breakdown fallback on the device (strategies.cpp:46-60).
//
// One CTA per broken-down group: LU with partial pivoting of the group's
// block-diagonal matrix (dense_lu.cpp:18-63: max magnitude, ties to the lowest
// row; rows physically swapped here, addressed through perm[] there -- the
// values are the same), blocked in column panels, forward and backward
// substitution in the reference's summation order, then the fallback residual
// through the group's reduction plan (one interval, or block_width-wide
// intervals + sequential combine for Multi-cells).
//
// Two modes.
//  * Dense (mode 1, and every one-cell group): densify the whole group
//    (dense_lu.cpp:8-16) and factor it, exactly the reference's arithmetic.
//  * Block-diagonal (mode 0, groups of k > 1 cells): the reference densifies a
//    k-cell group into a (k*s)^2 matrix whose off-diagonal blocks are zero and
//    runs the O((k*s)^3) LU over it.  With finite values every cross-block
//    operation is `a - (+-0)` or `(+-0) * finite`, which leaves nonzero values
//    unchanged and can only flip the SIGN OF A ZERO.  This mode factors the k
//    diagonal blocks one after another (k^2 times less work) and replays those
//    sign effects exactly:
//      - factorization: a -0 entry of block c becomes +0 iff some pivot of an
//        earlier block is negative (the update subtracts l*u = (+0/pivot)*(+0));
//      - forward (j ascending, earlier blocks first): a row whose right-hand
//        side is -0 becomes +0 iff some earlier column j has
//        signbit(pivot_j) != signbit(y_j) (the product (+0/pivot_j)*y_j is -0);
//      - backward (j ascending, in-block first): a row whose in-block sum is -0
//        becomes +0 iff some later x_j has its sign bit set ((+0)*x_j is -0).
//    Any non-finite input or result (where 0*inf = NaN would spread across
//    blocks) reports status 2 and the host reruns that group in dense mode.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bc {

struct LuEntry {
    int64_t cell0;  // first cell of the group
    int64_t gout;   // output group index
    int32_t kc;     // cells in the group
    int32_t pad;
};

struct LuParams {
    const double* values;
    const double* rhs;
    double* x_out;
    double* g_rms;
    int32_t* status;  // per entry: 0 ok, 1 singular, 2 non-finite (mode 0: rerun dense)
    const LuEntry* entries;
    const int32_t* row_ptr;  // pattern (device)
    const int32_t* col_idx;
    double* scratch;         // per entry: `stride` doubles
    int64_t stride;          // dense: n_max^2; block-diagonal: k_max * s^2
    int species, nnz;
    int block_width;         // 0 = single interval
    int mode;                // 0 block-diagonal when k > 1, 1 dense
    int panel_rows;          // > 0: panels are factored in shared memory (rows <= panel_rows)
    int smem_block;          // block-diagonal mode: each s x s block is densified, factored and
                             // forward-substituted in shared memory, then parked in scratch
                             // for the backward pass (one CTA per SM; 156^2 doubles = 195 KB)
    // dense mode, cells as links of a longer block-diagonal chain (Multi-cells
    // systems too large to densify, solved cell by cell): the three sign-of-
    // zero rules applied to this cell, and its flags for the host's chain scan
    int conv, flip, later_neg;
    uint8_t* chain_flags;    // per entry, or null: kChain* bits
};

constexpr uint8_t kChainNegPivot = 1;     // some pivot is negative
constexpr uint8_t kChainNegZeroVal = 2;   // some matrix value is -0
constexpr uint8_t kChainFwd = 4;          // some signbit(pivot_j) != signbit(y_j)
constexpr uint8_t kChainNegZeroRhs = 8;   // some right-hand side entry is -0
constexpr uint8_t kChainBwd = 16;         // some x has its sign bit set
constexpr uint8_t kChainNegZeroSum = 32;  // some backward row summed to -0

__device__ __forceinline__ void lu_argmax_combine(double& m, int& i, double m2, int i2) {
    // larger magnitude wins; equal magnitude -> lower row (strict > scan)
    if (m2 > m || (m2 == m && i2 < i)) {
        m = m2;
        i = i2;
    }
}

__device__ __forceinline__ bool is_neg_zero(double v) { return v == 0.0 && signbit(v); }

// Right-looking LU in panels of kLuPanel columns on physically swapped rows:
// every element still receives its updates a_ij -= l_ik * u_kj one k at a
// time in ascending k, each product and difference rounded separately, with
// the operands the reference's unblocked loop uses -- so the factors are bit-
// identical -- but the trailing matrix is read and written once per panel
// instead of once per k (K-fold less L2/HBM traffic), in 64x64 tiles whose
// L and U panels are staged in shared memory.
constexpr int kLuPanel = 16;
constexpr int kLuTile = 64;  // A22 tile edge: 256 threads x (4 x 4) register micro-tiles

// Factor the n x n row-major matrix `lu` in place (all threads of the CTA);
// perm[] (shared) starts as the identity and records the row swaps.  Returns
// false when the matrix is exactly singular (dense_lu.cpp:35).
// Panel of columns [k0, k1) factored by the whole CTA in shared memory (pbuf:
// rows [k0, n) x kLuPanel + 1, one row per thread per pass): the same pivot
// choice and per-element update order as the unblocked loop in lu_factor,
// three barriers per column.  Every thread combines the eight warp winners
// itself, so the pivot needs no broadcast.  Row swaps are applied to the
// panel here and to the other columns afterwards (nothing else reads them in
// between).  Returns false (uniformly) if singular.
__device__ bool lu_panel_cta(const int n, int* perm, double* pbuf, const int k0, const int k1, int* piv_out,
                             double* red_m, int* red_i) {
    constexpr int LD = kLuPanel + 1;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid % 32, warp = tid / 32, nw = nt / 32;
    const int K = k1 - k0, rows = n - k0;
    for (int kk = 0; kk < K; ++kk) {
        // dense_lu.cpp:32-41: largest magnitude in column k, ties to the lowest row
        const double a0 = fabs(pbuf[kk * LD + kk]);
        double bm = -1.0;
        int bi = n;
        if (isnan(a0)) {  // every later comparison with NaN fails: pivot stays k (uniform branch)
            bm = a0;
            bi = kk;
        } else {
            for (int r = kk + tid; r < rows; r += nt) {
                const double mag = fabs(pbuf[r * LD + kk]);
                if (!isnan(mag)) lu_argmax_combine(bm, bi, mag, r);
            }
            for (int off = 16; off >= 1; off >>= 1) {
                const double m2 = __shfl_xor_sync(0xffffffffu, bm, off);
                const int i2 = __shfl_xor_sync(0xffffffffu, bi, off);
                lu_argmax_combine(bm, bi, m2, i2);
            }
            if (lane == 0) {
                red_m[warp] = bm;
                red_i[warp] = bi;
            }
            __syncthreads();
            bm = red_m[0];
            bi = red_i[0];
            for (int w = 1; w < nw; ++w) lu_argmax_combine(bm, bi, red_m[w], red_i[w]);
        }
        if (bm == 0.0) return false;  // dense_lu.cpp:35 (every thread sees the same bm)
        if (tid == 0) {
            piv_out[kk] = k0 + bi;
            const int t = perm[k0 + kk];
            perm[k0 + kk] = perm[k0 + bi];
            perm[k0 + bi] = t;
        }
        if (bi != kk && tid < K) {
            const double t = pbuf[kk * LD + tid];
            pbuf[kk * LD + tid] = pbuf[bi * LD + tid];
            pbuf[bi * LD + tid] = t;
        }
        __syncthreads();
        // l_rk = a_rk / pivot, then row r's rest of the panel
        const double pv = pbuf[kk * LD + kk];
        for (int r = kk + 1 + tid; r < rows; r += nt) {
            double* row = pbuf + r * LD;
            const double l = __ddiv_rn(row[kk], pv);
            row[kk] = l;
#pragma unroll
            for (int c = 0; c < kLuPanel; ++c)
                if (c > kk && c < K) row[c] = __dsub_rn(row[c], __dmul_rn(l, pbuf[kk * LD + c]));
        }
        __syncthreads();
    }
    return true;  // the CTA writes pbuf back (lu_factor)
}

__device__ bool lu_factor(double* lu, const int n, int* perm, double* pbuf) {
    __shared__ double red_m[8];
    __shared__ int red_i[8];
    __shared__ int s_pivot, s_singular;
    __shared__ double s_lt[kLuTile][kLuPanel + 1];  // L21 tile (rows x panel)
    __shared__ double s_ut[kLuPanel][kLuTile];      // U12 tile (panel x cols)
    static_assert(kLuTile == 64, "the A22 micro-tiling below assumes 256 threads on a 64 x 64 tile");
    const int tid = threadIdx.x, nt = blockDim.x;
    // n <= 2048 (kMaxGroupRows): 32-bit element offsets
    auto A = [&](int i, int j) -> double& { return lu[i * n + j]; };
    if (tid == 0) s_singular = 0;
    __syncthreads();

    __shared__ int s_piv[kLuPanel];
    for (int k0 = 0; k0 < n; k0 += kLuPanel) {
        const int k1 = min(n, k0 + kLuPanel);
        if (pbuf) {
            // the panel (rows [k0, n) x columns [k0, k1)) into shared memory by the
            // whole CTA -- warp 0 alone would expose one L2 round trip per row
            {
                const int K = k1 - k0, rows = n - k0;
                for (int q = tid; q < rows * K; q += nt) {
                    const int r = q / K, c = q % K;
                    pbuf[r * (kLuPanel + 1) + c] = A(k0 + r, k0 + c);
                }
            }
            __syncthreads();
            if (!lu_panel_cta(n, perm, pbuf, k0, k1, s_piv, red_m, red_i)) return false;
            {
                const int K = k1 - k0, rows = n - k0;
                for (int q = tid; q < rows * K; q += nt) {
                    const int r = q / K, c = q % K;
                    A(k0 + r, k0 + c) = pbuf[r * (kLuPanel + 1) + c];
                }
            }
            // the panel's row swaps, in order, on the columns outside it
            for (int c = tid; c < n; c += nt) {
                if (c >= k0 && c < k1) continue;
                for (int kk = 0; kk < k1 - k0; ++kk) {
                    const int pr = s_piv[kk];
                    if (pr != k0 + kk) {
                        const double t = A(k0 + kk, c);
                        A(k0 + kk, c) = A(pr, c);
                        A(pr, c) = t;
                    }
                }
            }
            __syncthreads();
        }
        // panel factorization: columns [k0, k1), rows [k0, n)
        for (int k = k0; k < (pbuf ? k0 : k1); ++k) {
            // dense_lu.cpp:32-41: largest magnitude in column k, ties to the lowest row
            const double a0 = fabs(A(k, k));
            double bm = -1.0;
            int bi = n;
            if (isnan(a0)) {
                bm = a0;  // every later comparison with NaN fails: pivot stays k
                bi = k;
            } else {
                for (int i = k + tid; i < n; i += nt) {
                    const double mag = fabs(A(i, k));
                    if (!isnan(mag)) lu_argmax_combine(bm, bi, mag, i);
                }
                for (int off = 16; off >= 1; off >>= 1) {
                    const double m2 = __shfl_down_sync(0xffffffffu, bm, off);
                    const int i2 = __shfl_down_sync(0xffffffffu, bi, off);
                    lu_argmax_combine(bm, bi, m2, i2);
                }
                if ((tid & 31) == 0) {
                    red_m[tid >> 5] = bm;
                    red_i[tid >> 5] = bi;
                }
            }
            __syncthreads();
            if (tid == 0) {
                if (!isnan(a0)) {
                    bm = red_m[0];
                    bi = red_i[0];
                    for (int w = 1; w < nt / 32; ++w) lu_argmax_combine(bm, bi, red_m[w], red_i[w]);
                }
                if (bm == 0.0) s_singular = 1;  // dense_lu.cpp:35
                s_pivot = bi;
                const int t = perm[k];
                perm[k] = perm[bi];
                perm[bi] = t;
            }
            __syncthreads();
            if (s_singular) return false;
            const int piv = s_pivot;
            if (piv != k)  // the whole row moves (its trailing part is as stale as row k's)
                for (int c = tid; c < n; c += nt) {
                    const double t = A(k, c);
                    A(k, c) = A(piv, c);
                    A(piv, c) = t;
                }
            __syncthreads();
            const double pv = A(k, k);
            for (int i = k + 1 + tid; i < n; i += nt) A(i, k) = __ddiv_rn(A(i, k), pv);
            __syncthreads();
            const int w = k1 - k - 1;  // the rest of the panel
            if (w > 0) {
                for (int64_t idx = tid; idx < static_cast<int64_t>(n - k - 1) * w; idx += nt) {
                    const int i = k + 1 + static_cast<int>(idx / w), j = k + 1 + static_cast<int>(idx % w);
                    A(i, j) = __dsub_rn(A(i, j), __dmul_rn(A(i, k), A(k, j)));
                }
                __syncthreads();
            }
        }
        if (k1 == n) break;
        // U12: rows [k0, k1), columns [k1, n): a_ij -= l_ik u_kj for k = k0 .. i-1,
        // one column per thread held in registers (L11 from the panel buffer)
        {
            const int K = k1 - k0;
            for (int j = k1 + tid; j < n; j += nt) {
                double u[kLuPanel];
#pragma unroll
                for (int i = 0; i < kLuPanel; ++i) u[i] = i < K ? A(k0 + i, j) : 0.0;
#pragma unroll
                for (int k = 0; k < kLuPanel; ++k)
#pragma unroll
                    for (int i = k + 1; i < kLuPanel; ++i)
                        if (i < K) {
                            const double l = pbuf ? pbuf[i * (kLuPanel + 1) + k] : A(k0 + i, k0 + k);
                            u[i] = __dsub_rn(u[i], __dmul_rn(l, u[k]));
                        }
#pragma unroll
                for (int i = 1; i < kLuPanel; ++i)
                    if (i < K) A(k0 + i, j) = u[i];
            }
        }
        __syncthreads();
        // A22: rows and columns [k1, n), the panel's updates in ascending k per element
        const int K = k1 - k0, m = n - k1, tiles = (m + kLuTile - 1) / kLuTile;
        for (int t = 0; t < tiles * tiles; ++t) {
            const int i0 = k1 + (t / tiles) * kLuTile, j0 = k1 + (t % tiles) * kLuTile;
            for (int q = tid; q < kLuTile * kLuPanel; q += nt) {
                const int r = q / kLuPanel, kk = q % kLuPanel;
                s_lt[r][kk] = (i0 + r < n && kk < K) ? A(i0 + r, k0 + kk) : 0.0;
                const int kr = q / kLuTile, c = q % kLuTile;
                s_ut[kr][c] = (j0 + c < n && kr < K) ? A(k0 + kr, j0 + c) : 0.0;
            }
            __syncthreads();
            // thread (tr, tc) owns rows 4tr..4tr+3 and columns tc + 16q of the tile; per
            // element the panel's updates still run one k at a time in ascending order
            const int tr = tid / 16, tc = tid % 16;
            const bool interior = i0 + kLuTile <= n && j0 + kLuTile <= n;
            if (tid < 256) {
                double a[4][4];
                if (interior) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int q = 0; q < 4; ++q) a[i][q] = A(i0 + 4 * tr + i, j0 + tc + 16 * q);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int r = i0 + 4 * tr + i, cc = j0 + tc + 16 * q;
                            a[i][q] = (r < n && cc < n) ? A(r, cc) : 0.0;
                        }
                }
                for (int kk = 0; kk < K; ++kk) {
                    double l[4], u[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) l[i] = s_lt[4 * tr + i][kk];
#pragma unroll
                    for (int q = 0; q < 4; ++q) u[q] = s_ut[kk][tc + 16 * q];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int q = 0; q < 4; ++q) a[i][q] = __dsub_rn(a[i][q], __dmul_rn(l[i], u[q]));
                }
                if (interior) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int q = 0; q < 4; ++q) A(i0 + 4 * tr + i, j0 + tc + 16 * q) = a[i][q];
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int r = i0 + 4 * tr + i, cc = j0 + tc + 16 * q;
                            if (r < n && cc < n) A(r, cc) = a[i][q];
                        }
                }
            }
            __syncthreads();
        }
    }
    return true;
}

// Forward substitution L y = P b (dense_lu.cpp:53-57) on y[] (shared, holding
// P b): row i subtracts j = 0..i-1 in order, as a wavefront over j.  Each
// thread's row entries l_ij are read kLuFwdAhead steps ahead of use, so the
// per-step cost is the barrier, not an L2 round trip.
constexpr int kLuFwdAhead = 8;
__device__ void lu_forward(const double* lu, const int n, double* y) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (n <= nt) {  // one row per thread (every block-diagonal block and most groups)
        const int i = tid;
        const double* row = lu + static_cast<int64_t>(i < n ? i : 0) * n;
        double win[kLuFwdAhead];
#pragma unroll
        for (int q = 0; q < kLuFwdAhead; ++q) win[q] = (i < n && q < i) ? row[q] : 0.0;
        for (int j0 = 0; j0 < n; j0 += kLuFwdAhead) {
            double nxt[kLuFwdAhead];
#pragma unroll
            for (int q = 0; q < kLuFwdAhead; ++q) {
                const int j = j0 + kLuFwdAhead + q;
                nxt[q] = (i < n && j < i) ? row[j] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kLuFwdAhead; ++q) {
                const int j = j0 + q;
                __syncthreads();
                if (j < n && i > j && i < n) y[i] = __dsub_rn(y[i], __dmul_rn(win[q], y[j]));
            }
#pragma unroll
            for (int q = 0; q < kLuFwdAhead; ++q) win[q] = nxt[q];
        }
        __syncthreads();
        return;
    }
    for (int j = 0; j < n; ++j) {
        __syncthreads();
        const double xj = y[j];
        for (int i = j + 1 + tid; i < n; i += nt)
            y[i] = __dsub_rn(y[i], __dmul_rn(lu[static_cast<int64_t>(i) * n + j], xj));
    }
    __syncthreads();
}

// Backward substitution U x = y (dense_lu.cpp:58-62) in place on x[]: row ii
// subtracts j = ii+1..n-1 in order.  later_neg: a -0 sum turns +0 before the
// division (block-diagonal mode: the zero products of later blocks, see top).
// The row sums form one dependent chain, so warp 0 alone runs it (lanes form
// the products, lane 0 the ordered sum) with warp-level syncs only.
__device__ bool lu_backward(const double* lu, const int n, double* x, double* slots, const bool later_neg) {
    __shared__ int s_negzero_sum;
    const int tid = threadIdx.x;
    if (tid < 32) {
        // lane L owns columns j = L + 32q; the next row's entries (and its
        // pivot, for lane 0) are loaded while lane 0 runs this row's chain
        const int nq = (n + 31) / 32;  // columns per lane
        bool z = false;
        double cur[8], nxt[8], dcur = 0.0, dnxt = 0.0;
        auto load_row = [&](int ii, double (&dst)[8], double& dg) {
            const double* row = lu + static_cast<int64_t>(ii) * n;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int j = tid + 32 * q;
                dst[q] = (q < nq && j > ii && j < n) ? row[j] : 0.0;
            }
            dg = tid == 0 ? row[ii] : 0.0;
        };
        if (nq <= 8) {
            load_row(n - 1, cur, dcur);
            for (int ii = n - 1; ii >= 0; --ii) {
                if (ii > 0) load_row(ii - 1, nxt, dnxt);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int j = tid + 32 * q;
                    if (q < nq && j > ii && j < n) slots[j] = __dmul_rn(cur[q], x[j]);
                }
                __syncwarp();
                if (tid == 0) {
                    double acc = x[ii];
#pragma unroll 8
                    for (int j = ii + 1; j < n; ++j) acc = __dsub_rn(acc, slots[j]);
                    if (is_neg_zero(acc)) {
                        z = true;
                        if (later_neg) acc = 0.0;
                    }
                    x[ii] = __ddiv_rn(acc, dcur);
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
                dcur = dnxt;
            }
        } else {
            for (int ii = n - 1; ii >= 0; --ii) {
                const double* row = lu + static_cast<int64_t>(ii) * n;
                for (int j = ii + 1 + tid; j < n; j += 32) slots[j] = __dmul_rn(row[j], x[j]);
                __syncwarp();
                if (tid == 0) {
                    double acc = x[ii];
#pragma unroll 8
                    for (int j = ii + 1; j < n; ++j) acc = __dsub_rn(acc, slots[j]);
                    if (is_neg_zero(acc)) {
                        z = true;
                        if (later_neg) acc = 0.0;
                    }
                    x[ii] = __ddiv_rn(acc, row[ii]);
                }
                __syncwarp();
            }
        }
        if (tid == 0) s_negzero_sum = z;
    }
    __syncthreads();
    return s_negzero_sum != 0;
}

// lu_backward for one warp (any warp of the CTA) on one block, with the
// block's own product slots: returns (warp-uniform) whether some row summed
// to -0 -- the case where a later block's negative x would have flipped it
// (block-diagonal mode runs every block's chain at once with later_neg
// false, then redoes the rare blocks where that guess was wrong).
__device__ bool lu_backward_warp(const double* lu, const int n, double* x, double* slots, const bool later_neg) {
    const int lane = threadIdx.x % 32;
    const int nq = (n + 31) / 32;
    bool z = false;
    double cur[8], nxt[8], dcur = 0.0, dnxt = 0.0;
    auto load_row = [&](int ii, double (&dst)[8], double& dg) {
        const double* row = lu + static_cast<int64_t>(ii) * n;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int j = lane + 32 * q;
            dst[q] = (q < nq && j > ii && j < n) ? row[j] : 0.0;
        }
        dg = lane == 0 ? row[ii] : 0.0;
    };
    if (nq > 8) {  // rows longer than 256: no prefetch window, the plain loop
        for (int ii = n - 1; ii >= 0; --ii) {
            const double* row = lu + static_cast<int64_t>(ii) * n;
            for (int j = ii + 1 + lane; j < n; j += 32) slots[j] = __dmul_rn(row[j], x[j]);
            __syncwarp();
            if (lane == 0) {
                double acc = x[ii];
#pragma unroll 8
                for (int j = ii + 1; j < n; ++j) acc = __dsub_rn(acc, slots[j]);
                if (is_neg_zero(acc)) {
                    z = true;
                    if (later_neg) acc = 0.0;
                }
                x[ii] = __ddiv_rn(acc, row[ii]);
            }
            __syncwarp();
        }
        return __shfl_sync(0xffffffffu, z ? 1 : 0, 0) != 0;
    }
    load_row(n - 1, cur, dcur);
    for (int ii = n - 1; ii >= 0; --ii) {
        if (ii > 0) load_row(ii - 1, nxt, dnxt);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int j = lane + 32 * q;
            if (q < nq && j > ii && j < n) slots[j] = __dmul_rn(cur[q], x[j]);
        }
        __syncwarp();
        if (lane == 0) {
            double acc = x[ii];
#pragma unroll 8
            for (int j = ii + 1; j < n; ++j) acc = __dsub_rn(acc, slots[j]);
            if (is_neg_zero(acc)) {
                z = true;
                if (later_neg) acc = 0.0;
            }
            x[ii] = __ddiv_rn(acc, dcur);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
        dcur = dnxt;
    }
    return __shfl_sync(0xffffffffu, z ? 1 : 0, 0) != 0;
}

// Scatter cells [c0, c0 + cells) of the group into the zeroed dense matrix
// `lu` (row length ld): dense_lu.cpp:8-16 on the block-diagonal matrix.
__device__ void lu_densify(double* lu, const int ld, const double* vals, const int32_t* row_ptr,
                           const int32_t* col_idx, const int s, const int nnz, const int cells) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int n = cells * s;
    for (int64_t idx = tid; idx < static_cast<int64_t>(n) * ld; idx += nt) lu[idx] = 0.0;
    __syncthreads();
    for (int i = tid; i < n; i += nt) {
        const int c = i / s, r = i % s;
        for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e)
            lu[static_cast<int64_t>(i) * ld + (ld == s ? 0 : c * s) + col_idx[e]] = vals[c * nnz + e];
    }
    __syncthreads();
}

// The residual of a group's fallback solution x (shared) through the group's
// reduction plan (strategies.cpp:48-58; spmv csr.cpp:90-101; plan_reduce_map
// reduction.hpp:60-79) into g_rms, and status 0.  All threads of the CTA.
__device__ void lu_group_residual(const LuParams& p, const LuEntry& ent, const int n, const double* vals,
                                  const double* b, const double* x, double* slots) {
    const int tid = threadIdx.x, nt = blockDim.x, s = p.species;
    const int width = p.block_width > 0 ? p.block_width : n;
    double total = 0.0;
    for (int b0 = 0, blk = 0; b0 < n; b0 += width, ++blk) {
        const int len = min(width, n - b0);
        int P = 1;
        while (P < len) P <<= 1;
        __syncthreads();
        for (int q = tid; q < P; q += nt) {
            double v = 0.0;
            if (q < len) {
                const int i = b0 + q, c = i / s, r = i % s;
                double acc = 0.0;
                for (int e = p.row_ptr[r]; e < p.row_ptr[r + 1]; ++e)
                    acc = __dadd_rn(acc, __dmul_rn(vals[c * p.nnz + e], x[c * s + p.col_idx[e]]));
                const double ri = __dsub_rn(b[i], acc);
                v = __dmul_rn(ri, ri);
            }
            slots[q] = v;
        }
        for (int stride = P / 2; stride >= 1; stride /= 2) {
            __syncthreads();
            for (int q = tid; q < stride; q += nt) slots[q] = __dadd_rn(slots[q], slots[q + stride]);
        }
        __syncthreads();
        total = blk == 0 ? slots[0] : __dadd_rn(total, slots[0]);
    }
    if (tid == 0) {
        p.g_rms[ent.gout] = __dsqrt_rn(__ddiv_rn(total, static_cast<double>(n)));
        p.status[blockIdx.x] = 0;
    }
}

__global__ void __launch_bounds__(256, 3) lu_fallback_kernel(const LuParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const LuEntry ent = p.entries[blockIdx.x];
    const int s = p.species;
    const int n = ent.kc * s;
    double* lu = p.scratch + static_cast<size_t>(blockIdx.x) * p.stride;
    // dynamic shared memory: [panel buffer] perm | sum | slots, or (smem_block)
    // perm | sum | the block being factored (also the slots, once every block is done)
    double* pbuf = nullptr;
    const int prow = p.mode == 0 && ent.kc > 1 ? s : n;
    unsigned char* base = smem_raw;
    if (p.panel_rows > 0 && !p.smem_block) {
        if (prow <= p.panel_rows) pbuf = reinterpret_cast<double*>(smem_raw);
        base += sizeof(double) * p.panel_rows * (kLuPanel + 1);
    }
    int* perm = reinterpret_cast<int*>(base);
    double* sum = reinterpret_cast<double*>(base + sizeof(int) * ((n + 1) & ~1));
    double* ycopy = sum + n;  // block-diagonal mode: the forward results, for the rare backward redo
    double* slots = ycopy + n;  // >= max(padded length, 8 * species) (also used for products)
    double* sblk = p.smem_block ? slots : nullptr;
    const int tid = threadIdx.x, nt = blockDim.x;
    const double* vals = p.values + ent.cell0 * p.nnz;
    const double* b = p.rhs + ent.cell0 * s;

    for (int i = tid; i < n; i += nt) perm[i] = i % (p.mode == 0 && ent.kc > 1 ? s : n);
    if (p.mode == 0 && ent.kc > 1) {
        // block-diagonal mode: finite inputs only
        int bad = 0;
        for (int64_t q = tid; q < static_cast<int64_t>(ent.kc) * p.nnz; q += nt) bad |= !isfinite(vals[q]);
        for (int q = tid; q < n; q += nt) bad |= !isfinite(b[q]);
        if (__syncthreads_or(bad)) {
            if (tid == 0) p.status[blockIdx.x] = 2;
            return;
        }
        bool neg_pivot = false, fwd_flip = false;
        for (int c = 0; c < ent.kc; ++c) {
            double* gblk = lu + static_cast<int64_t>(c) * s * s;
            double* blk = sblk ? sblk : gblk;
            lu_densify(blk, s, vals + static_cast<int64_t>(c) * p.nnz, p.row_ptr, p.col_idx, s, p.nnz, 1);
            if (neg_pivot)
                for (int q = tid; q < s * s; q += nt)
                    if (is_neg_zero(blk[q])) blk[q] = 0.0;
            __syncthreads();
            if (!lu_factor(blk, s, perm + c * s, pbuf)) {
                if (tid == 0) p.status[blockIdx.x] = 1;
                return;
            }
            int neg = 0, nonfinite = 0;
            for (int q = tid; q < s * s; q += nt) nonfinite |= !isfinite(blk[q]);
            for (int i = tid; i < s; i += nt) neg |= signbit(blk[i * s + i]) ? 1 : 0;
            neg_pivot = __syncthreads_or(neg) || neg_pivot;
            if (__syncthreads_or(nonfinite)) {
                if (tid == 0) p.status[blockIdx.x] = 2;
                return;
            }
            double* y = sum + c * s;
            for (int i = tid; i < s; i += nt) {
                double v = b[c * s + perm[c * s + i]];
                if (fwd_flip && is_neg_zero(v)) v = 0.0;
                y[i] = v;
            }
            lu_forward(blk, s, y);
            int flip = 0;
            for (int i = tid; i < s; i += nt) flip |= (signbit(blk[i * s + i]) != signbit(y[i])) ? 1 : 0;
            fwd_flip = __syncthreads_or(flip) || fwd_flip;
            if (sblk)  // park the factors for the backward pass (the next block reuses the buffer)
                for (int q = tid; q < s * s; q += nt) gblk[q] = sblk[q];
            __syncthreads();
        }
        // Backward substitutions of all blocks at once, one warp per block, each
        // assuming no later block has a negative x (later_neg false); then, in
        // the reference's order (last block first), the rare block that summed a
        // row to -0 while a later x is negative is redone from its forward result.
        __shared__ unsigned s_zmask[64];  // kc <= kMaxGroupRows / 1
        for (int i = tid; i < 64; i += nt) s_zmask[i] = 0u;
        for (int i = tid; i < n; i += nt) ycopy[i] = sum[i];
        __syncthreads();
        {
            const int warp = tid / 32, nw = nt / 32;
            for (int c = warp; c < ent.kc; c += nw) {
                const bool z = lu_backward_warp(lu + static_cast<int64_t>(c) * s * s, s, sum + c * s,
                                                slots + warp * s, false);
                if (z && (tid % 32) == 0) atomicOr(&s_zmask[c / 32], 1u << (c % 32));
            }
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
    } else {
        lu_densify(lu, n, vals, p.row_ptr, p.col_idx, s, p.nnz, ent.kc);
        int nzv = 0;
        for (int64_t q = tid; q < static_cast<int64_t>(ent.kc) * p.nnz; q += nt) nzv |= is_neg_zero(vals[q]);
        if (p.conv)
            for (int64_t q = tid; q < static_cast<int64_t>(n) * n; q += nt)
                if (is_neg_zero(lu[q])) lu[q] = 0.0;
        __syncthreads();
        if (!lu_factor(lu, n, perm, pbuf)) {
            if (tid == 0) p.status[blockIdx.x] = 1;
            return;
        }
        int nzb = 0;
        for (int i = tid; i < n; i += nt) {
            double v = b[perm[i]];
            nzb |= is_neg_zero(v);
            if (p.flip && is_neg_zero(v)) v = 0.0;
            sum[i] = v;
        }
        lu_forward(lu, n, sum);
        int neg = 0, fwd = 0;
        for (int i = tid; i < n; i += nt) {
            const double u = lu[static_cast<int64_t>(i) * n + i];
            neg |= signbit(u) ? 1 : 0;
            fwd |= signbit(u) != signbit(sum[i]) ? 1 : 0;
        }
        __syncthreads();  // the flags above read y before the back substitution overwrites it
        const bool z = lu_backward(lu, n, sum, slots, p.later_neg != 0);
        int bwd = 0;
        for (int i = tid; i < n; i += nt) bwd |= signbit(sum[i]) ? 1 : 0;
        const uint8_t fl = (__syncthreads_or(neg) ? kChainNegPivot : 0) | (__syncthreads_or(nzv) ? kChainNegZeroVal : 0) |
                           (__syncthreads_or(fwd) ? kChainFwd : 0) | (__syncthreads_or(nzb) ? kChainNegZeroRhs : 0) |
                           (__syncthreads_or(bwd) ? kChainBwd : 0) | (z ? kChainNegZeroSum : 0);
        if (p.chain_flags && tid == 0) p.chain_flags[blockIdx.x] = fl;
    }
    double* xo = p.x_out + ent.cell0 * s;
    for (int i = tid; i < n; i += nt) xo[i] = sum[i];

    lu_group_residual(p, ent, n, vals, b, sum, slots);
}

}  // namespace bc
