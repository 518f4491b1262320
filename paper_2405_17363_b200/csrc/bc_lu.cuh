// bc_lu.cuh -- breakdown fallback on the device (strategies.cpp:46-60).
//
// One CTA per broken-down group: densify the group's block-diagonal matrix
// (dense_lu.cpp:8-16), LU with partial pivoting -- max magnitude, ties to the
// lowest row, rows physically swapped (dense_lu.cpp:18-63 addresses them
// through perm[]; the values are the same), blocked in column panels -- forward
// and backward substitution in the reference's summation order, then the
// fallback residual through the group's reduction plan (one interval, or
// block_width-wide intervals + sequential combine for Multi-cells).
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
    int32_t* status;  // per entry: 0 ok, 1 singular
    const LuEntry* entries;
    const int32_t* row_ptr;  // pattern (device)
    const int32_t* col_idx;
    double* scratch;         // per entry: n_max * n_max
    int64_t n_max;
    int species, nnz;
    int block_width;         // 0 = single interval
};

__device__ __forceinline__ void lu_argmax_combine(double& m, int& i, double m2, int i2) {
    // larger magnitude wins; equal magnitude -> lower row (strict > scan)
    if (m2 > m || (m2 == m && i2 < i)) {
        m = m2;
        i = i2;
    }
}

// Right-looking LU in panels of kLuPanel columns on physically swapped rows:
// every element still receives its updates a_ij -= l_ik * u_kj one k at a
// time in ascending k, each product and difference rounded separately, with
// the operands the reference's unblocked loop uses -- so the factors are bit-
// identical -- but the trailing matrix is read and written once per panel
// instead of once per k (K-fold less L2/HBM traffic), in 32x32 tiles whose
// L and U panels are staged in shared memory.
constexpr int kLuPanel = 16;
constexpr int kLuTile = 64;  // A22 tile edge: 256 threads x (4 x 4) register micro-tiles

__global__ void __launch_bounds__(256) lu_fallback_kernel(const LuParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const LuEntry ent = p.entries[blockIdx.x];
    const int s = p.species;
    const int n = ent.kc * s;
    double* lu = p.scratch + static_cast<size_t>(blockIdx.x) * p.n_max * p.n_max;
    int* perm = reinterpret_cast<int*>(smem_raw);
    double* sum = reinterpret_cast<double*>(smem_raw + sizeof(int) * ((n + 1) & ~1));
    double* slots = sum + n;  // >= padded length (also used for products)
    __shared__ double red_m[8];
    __shared__ int red_i[8];
    __shared__ int s_pivot, s_singular;
    __shared__ double s_lt[kLuTile][kLuPanel + 1];  // L21 tile (rows x panel)
    __shared__ double s_ut[kLuPanel][kLuTile];      // U12 tile (panel x cols)
    static_assert(kLuTile == 64, "the A22 micro-tiling below assumes 256 threads on a 64 x 64 tile");
    const int tid = threadIdx.x, nt = blockDim.x;
    const double* vals = p.values + ent.cell0 * p.nnz;
    const double* b = p.rhs + ent.cell0 * s;
    auto A = [&](int i, int j) -> double& { return lu[static_cast<int64_t>(i) * n + j]; };

    // dense_lu.cpp:8-16 densify
    for (int64_t idx = tid; idx < static_cast<int64_t>(n) * n; idx += nt) lu[idx] = 0.0;
    __syncthreads();
    for (int i = tid; i < n; i += nt) {
        const int c = i / s, r = i % s;
        for (int e = p.row_ptr[r]; e < p.row_ptr[r + 1]; ++e) A(i, c * s + p.col_idx[e]) = vals[c * p.nnz + e];
        perm[i] = i;
    }
    if (tid == 0) s_singular = 0;
    __syncthreads();

    for (int k0 = 0; k0 < n; k0 += kLuPanel) {
        const int k1 = min(n, k0 + kLuPanel);
        // panel factorization: columns [k0, k1), rows [k0, n)
        for (int k = k0; k < k1; ++k) {
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
            if (s_singular) {
                if (tid == 0) p.status[blockIdx.x] = 1;
                return;
            }
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
        // U12: rows [k0, k1), columns [k1, n): a_ij -= l_ik u_kj for k = k0 .. i-1
        for (int j = k1 + tid; j < n; j += nt)
            for (int k = k0; k < k1; ++k) {
                const double ukj = A(k, j);
                for (int i = k + 1; i < k1; ++i) A(i, j) = __dsub_rn(A(i, j), __dmul_rn(A(i, k), ukj));
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
            if (tid < 256) {
                double a[4][4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int r = i0 + 4 * tr + i, cc = j0 + tc + 16 * q;
                        a[i][q] = (r < n && cc < n) ? A(r, cc) : 0.0;
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
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int r = i0 + 4 * tr + i, cc = j0 + tc + 16 * q;
                        if (r < n && cc < n) A(r, cc) = a[i][q];
                    }
            }
            __syncthreads();
        }
    }

    // forward: L y = P b, row i subtracts j = 0..i-1 in order (wavefront)
    for (int i = tid; i < n; i += nt) sum[i] = b[perm[i]];
    for (int j = 0; j < n; ++j) {
        __syncthreads();
        const double xj = sum[j];
        for (int i = j + 1 + tid; i < n; i += nt) sum[i] = __dsub_rn(sum[i], __dmul_rn(A(i, j), xj));
    }
    __syncthreads();
    // backward: U x = y, row ii subtracts j = ii+1..n-1 in order
    for (int ii = n - 1; ii >= 0; --ii) {
        for (int j = ii + 1 + tid; j < n; j += nt) slots[j] = __dmul_rn(A(ii, j), sum[j]);
        __syncthreads();
        if (tid == 0) {
            double acc = sum[ii];
            for (int j = ii + 1; j < n; ++j) acc = __dsub_rn(acc, slots[j]);
            sum[ii] = __ddiv_rn(acc, A(ii, ii));
        }
        __syncthreads();
    }
    double* xo = p.x_out + ent.cell0 * s;
    for (int i = tid; i < n; i += nt) xo[i] = sum[i];

    // residual of the fallback solution through the same plan
    // (strategies.cpp:48-58; spmv csr.cpp:90-101; plan_reduce_map reduction.hpp:60-79)
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
                    acc = __dadd_rn(acc, __dmul_rn(vals[c * p.nnz + e], sum[c * s + p.col_idx[e]]));
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

}  // namespace bc
