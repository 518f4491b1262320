// bc_thread.cuh -- one thread per cell (K4, comparison baseline; the
// "classic approach" of PAPER.md:43).
//
// Each thread runs a whole One-cell solve (strategies.cpp:158-174 semantics:
// one cell per group, reduction over next_pow2(species) slots).  Values and
// work vectors are cell-interleaved in global memory ([entry][cell]) so a warp's
// loads are coalesced; every iteration streams the cell's matrix and vectors
// through the memory hierarchy -- the streaming formulation the HBM roofline
// of SURVEY.md §8d describes.  Arithmetic is bit-identical to the reference:
// SpMV in CSR order, SpMV^T as the reference's row-ordered scatter, and each
// reduction evaluated as the same stride-halving tree, walked in order over
// bit-reversed leaf indices with a pairwise stack.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bc_block.cuh"

namespace bc {

struct ThreadParams {
    const double* values_il;  // nnz * cells (interleaved)
    const double* rhs;        // cells * species
    double* x_out;            // cells * species
    double* work;             // 9 * species * cells (interleaved)
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* diag;
    int32_t* g_iters;
    double* g_rms;
    uint8_t* g_flags;
    int64_t cells;
    int species, nnz, log2P;
    double tol;
    int64_t max_iter;
};

// transpose [cells][nnz] -> [nnz][cells]
__global__ void interleave_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t cells, int nnz) {
    __shared__ double tile[32][33];
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int e0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + k;
        const int e = e0 + threadIdx.x;
        if (c < cells && e < nnz) tile[k][threadIdx.x] = src[c * nnz + e];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int e = e0 + k;
        const int64_t c = c0 + threadIdx.x;
        if (c < cells && e < nnz) dst[static_cast<int64_t>(e) * cells + c] = tile[threadIdx.x][k];
    }
}

struct TpcView {
    const ThreadParams* p;
    int64_t c;
    __device__ __forceinline__ double a(int e) const { return p->values_il[static_cast<int64_t>(e) * p->cells + c]; }
    __device__ __forceinline__ double& w(int k, int i) const {
        return p->work[(static_cast<int64_t>(k) * p->species + i) * p->cells + c];
    }
};

__device__ __forceinline__ int bitrev(int t, int bits) { return bits ? static_cast<int>(__brev(t) >> (32 - bits)) : 0; }

// tree_reduce_in_place over next_pow2(n) slots, slot i = f(i) (0 beyond n)
template <class F>
__device__ double tpc_tree(int n, int log2P, F&& f) {
    double stack[13];
    const int P = 1 << log2P;
    for (int t = 0; t < P; ++t) {
        const int i = bitrev(t, log2P);
        double x = i < n ? f(i) : 0.0;
        int lvl = 0;
        while ((t >> lvl) & 1) {
            x = dadd(stack[lvl], x);
            ++lvl;
        }
        stack[lvl] = x;
    }
    return stack[log2P];
}

__device__ void tpc_spmv(const TpcView& v, int in, int out) {
    const ThreadParams& p = *v.p;
    for (int i = 0; i < p.species; ++i) {
        double acc = 0.0;
        for (int e = p.row_ptr[i]; e < p.row_ptr[i + 1]; ++e) acc = dadd(acc, dmul(v.a(e), v.w(in, p.col_idx[e])));
        v.w(out, i) = acc;
    }
}

__device__ void tpc_spmv_t(const TpcView& v, int in, int out) {  // csr.cpp:129-142
    const ThreadParams& p = *v.p;
    for (int j = 0; j < p.species; ++j) v.w(out, j) = 0.0;
    for (int i = 0; i < p.species; ++i) {
        const double xi = v.w(in, i);
        for (int e = p.row_ptr[i]; e < p.row_ptr[i + 1]; ++e) {
            double& y = v.w(out, p.col_idx[e]);
            y = dadd(y, dmul(v.a(e), xi));
        }
    }
}

template <int ALGO>
__global__ void __launch_bounds__(128) thread_per_cell_kernel(const ThreadParams p) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= p.cells) return;
    const TpcView v{&p, c};
    const int n = p.species;
    const double* b = p.rhs + c * n;
    // work vectors: 0 x, 1 r, 2 rh (r~), 3 p, 4 v (p~), 5 y/z (Ap), 6 t (A^T p~), 7 dinv, 8 Ax
    enum { X = 0, Rv = 1, RH = 2, PV = 3, V = 4, Y = 5, T = 6, D = 7, AX = 8 };
    auto fresh = [&]() {
        tpc_spmv(v, X, AX);
        const double sq = tpc_tree(n, p.log2P, [&](int i) {
            const double ri = dsub(b[i], v.w(AX, i));
            return dmul(ri, ri);
        });
        return __dsqrt_rn(ddiv(sq, static_cast<double>(n)));
    };
    for (int i = 0; i < n; ++i) v.w(X, i) = 0.0;
    tpc_spmv(v, X, AX);
    for (int i = 0; i < n; ++i) {
        const double ri = dadd(b[i], -v.w(AX, i));
        v.w(Rv, i) = ri;
        v.w(RH, i) = ri;
        if (ALGO == kBiCGStab) {
            v.w(PV, i) = 0.0;
            v.w(V, i) = 0.0;
            const int di = p.diag[i];
            const double d = di >= 0 ? v.a(di) : 0.0;
            v.w(D, i) = d != 0.0 ? ddiv(1.0, d) : 1.0;
        } else {
            v.w(PV, i) = ri;
            v.w(V, i) = ri;
        }
    }
    const double nd = static_cast<double>(n);
    double sigma = tpc_tree(n, p.log2P, [&](int i) { return dmul(v.w(Rv, i), v.w(Rv, i)); });
    int64_t iters = 0;
    bool conv = false, brk = false;
    double fres = 0.0;
    if (__dsqrt_rn(ddiv(sigma, nd)) <= p.tol) {
        fres = fresh();
        conv = fres <= p.tol;
    }
    if (!conv) {
        double rho_prev = ALGO == kBiCGStab ? 1.0 : 0.0, alpha = 1.0, omega = 1.0;
        for (int64_t it = 1; it <= p.max_iter; ++it) {
            const double rho = tpc_tree(n, p.log2P, [&](int i) { return dmul(v.w(RH, i), v.w(Rv, i)); });
            if (scalar_breaks(rho)) { brk = true; break; }
            if (ALGO == kBiCGStab) {
                const double beta = dmul(ddiv(rho, rho_prev), ddiv(alpha, omega));
                for (int i = 0; i < n; ++i) {
                    const double pi = dadd(v.w(Rv, i), dmul(beta, dsub(v.w(PV, i), dmul(omega, v.w(V, i)))));
                    v.w(PV, i) = pi;
                    v.w(Y, i) = dmul(v.w(D, i), pi);
                }
                tpc_spmv(v, Y, V);
                const double den = tpc_tree(n, p.log2P, [&](int i) { return dmul(v.w(RH, i), v.w(V, i)); });
                if (scalar_breaks(den)) { brk = true; break; }
                alpha = ddiv(rho, den);
                for (int i = 0; i < n; ++i) {
                    const double si = dsub(v.w(Rv, i), dmul(alpha, v.w(V, i)));
                    v.w(X, i) = dadd(v.w(X, i), dmul(alpha, v.w(Y, i)));
                    v.w(Rv, i) = si;
                    v.w(Y, i) = dmul(v.w(D, i), si);  // y <- z
                }
                tpc_spmv(v, Y, T);
                const double tt = tpc_tree(n, p.log2P, [&](int i) { return dmul(v.w(T, i), v.w(T, i)); });
                const double ts = tpc_tree(n, p.log2P, [&](int i) { return dmul(v.w(T, i), v.w(Rv, i)); });
                if (tt != 0.0 && scalar_breaks(tt)) { brk = true; break; }
                omega = tt == 0.0 ? 0.0 : ddiv(ts, tt);
                for (int i = 0; i < n; ++i) {
                    v.w(X, i) = dadd(v.w(X, i), dmul(omega, v.w(Y, i)));
                    v.w(Rv, i) = dsub(v.w(Rv, i), dmul(omega, v.w(T, i)));
                }
            } else {
                if (it > 1) {
                    const double beta = ddiv(rho, rho_prev);
                    for (int i = 0; i < n; ++i) {
                        v.w(PV, i) = dadd(v.w(Rv, i), dmul(beta, v.w(PV, i)));
                        v.w(V, i) = dadd(v.w(RH, i), dmul(beta, v.w(V, i)));
                    }
                }
                tpc_spmv(v, PV, Y);
                tpc_spmv_t(v, V, T);
                const double den = tpc_tree(n, p.log2P, [&](int i) { return dmul(v.w(V, i), v.w(Y, i)); });
                if (scalar_breaks(den)) { brk = true; break; }
                alpha = ddiv(rho, den);
                const double na = -alpha;
                for (int i = 0; i < n; ++i) {
                    v.w(X, i) = dadd(v.w(X, i), dmul(alpha, v.w(PV, i)));
                    v.w(Rv, i) = dadd(v.w(Rv, i), dmul(na, v.w(Y, i)));
                    v.w(RH, i) = dadd(v.w(RH, i), dmul(na, v.w(T, i)));
                }
            }
            rho_prev = rho;
            iters = it;
            sigma = tpc_tree(n, p.log2P, [&](int i) { return dmul(v.w(Rv, i), v.w(Rv, i)); });
            if (!isfinite(sigma)) { brk = true; break; }
            if (__dsqrt_rn(ddiv(sigma, nd)) <= p.tol) {
                const double f = fresh();
                if (f <= p.tol) {
                    fres = f;
                    conv = true;
                    break;
                }
            }
            if (ALGO == kBiCGStab && scalar_breaks(omega)) { brk = true; break; }
        }
        if (!conv) {
            fres = fresh();
            conv = !brk && fres <= p.tol;
        }
    }
    double* xo = p.x_out + c * n;
    for (int i = 0; i < n; ++i) xo[i] = v.w(X, i);
    p.g_iters[c] = static_cast<int32_t>(iters);
    p.g_rms[c] = fres;
    p.g_flags[c] = static_cast<uint8_t>((conv ? 1 : 0) | (brk ? 2 : 0));
}

}  // namespace bc
