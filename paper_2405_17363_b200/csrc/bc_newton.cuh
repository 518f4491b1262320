// bc_newton.cuh -- device Newton-system assembly.
//
// One thread per cell replays the reference's accumulation order exactly:
// rhs_into (mechanism.cpp:235-247), jacobian_into (mechanism.cpp:249-267)
// and fill_newton_system (simulate.cpp:37-41).  Rate constants come from
// the host (std::pow, mechanism.cpp:221-233), so values are bit-identical
// to the host generator.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bc {

struct NewtonParams {
    int64_t count;
    int species, reactions, nnz;
    const double* rates;  // count * reactions
    const int32_t *stamp_ptr, *stamp_slot, *stamp_other;
    const double* stamp_sign;
    const int32_t *reactant_ptr, *reactants, *product_ptr, *products, *diag_slot;
    double h;
    const double* y;       // count * species or nullptr (ones)
    const double* y_prev;  // count * species or nullptr (= y)
    double* values;        // count * nnz
    double* rhs;           // count * species
    double* f_scratch;     // count * species
};

__global__ void __launch_bounds__(128) newton_assemble_kernel(const NewtonParams p) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= p.count) return;
    const int s = p.species;
    const double* rates = p.rates + c * p.reactions;
    const double* y = p.y ? p.y + c * s : nullptr;
    const double* yp = p.y_prev ? p.y_prev + c * s : y;
    double* f = p.f_scratch + c * s;
    double* v = p.values + c * p.nnz;
    for (int i = 0; i < s; ++i) f[i] = 0.0;
    for (int j = 0; j < p.reactions; ++j) {
        double rate = rates[j];
        for (int q = p.reactant_ptr[j]; q < p.reactant_ptr[j + 1]; ++q)
            rate = __dmul_rn(rate, y ? y[p.reactants[q]] : 1.0);
        for (int q = p.reactant_ptr[j]; q < p.reactant_ptr[j + 1]; ++q)
            f[p.reactants[q]] = __dsub_rn(f[p.reactants[q]], rate);
        for (int q = p.product_ptr[j]; q < p.product_ptr[j + 1]; ++q)
            f[p.products[q]] = __dadd_rn(f[p.products[q]], rate);
    }
    for (int k = 0; k < p.nnz; ++k) v[k] = 0.0;
    for (int j = 0; j < p.reactions; ++j) {
        for (int q = p.stamp_ptr[j]; q < p.stamp_ptr[j + 1]; ++q) {
            double partial = rates[j];
            const int o = p.stamp_other[q];
            if (o >= 0) partial = __dmul_rn(partial, y ? y[o] : 1.0);
            v[p.stamp_slot[q]] = __dadd_rn(v[p.stamp_slot[q]], __dmul_rn(p.stamp_sign[q], partial));
        }
    }
    const double nh = -p.h;
    for (int k = 0; k < p.nnz; ++k) v[k] = __dmul_rn(nh, v[k]);
    for (int i = 0; i < s; ++i) v[p.diag_slot[i]] = __dadd_rn(v[p.diag_slot[i]], 1.0);
    double* b = p.rhs + c * s;
    for (int i = 0; i < s; ++i) {
        const double yi = y ? y[i] : 1.0;
        const double ypi = yp ? yp[i] : 1.0;
        b[i] = -__dsub_rn(__dsub_rn(yi, ypi), __dmul_rn(p.h, f[i]));
    }
}

// Newton update of the device-resident simulation (simulate.cpp:139-165):
// y += dy for every species of every cell, then max |dy| (update_inf) and
// max |y| (state_inf) over the batch and a count of non-finite states.  The
// host loop's `m = std::max(m, std::abs(v))` keeps m when v is NaN; the
// `m < |v|` test below does the same.  max is exact and order-free, so the
// block/atomic reduction is bit-equal to the host loop.  Non-negative
// doubles order like their bit patterns: atomicMax on the 64-bit words.
struct UpdateParams {
    int64_t n;                // cells * species
    double* y;
    const double* dy;
    unsigned long long* red;  // [0] update_inf bits, [1] state_inf bits, [2] non-finite count
};

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, v, m);
        if (v < o) v = o;
    }
    return v;
}

__global__ void __launch_bounds__(256) newton_update_kernel(const UpdateParams p) {
    __shared__ double s_u[8], s_s[8];
    __shared__ unsigned int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    double mu = 0.0, ms = 0.0;
    unsigned int bad = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < p.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double d = p.dy[i];
        const double ad = fabs(d);
        if (mu < ad) mu = ad;
        const double v = __dadd_rn(p.y[i], d);
        p.y[i] = v;
        if (!isfinite(v)) ++bad;
        const double av = fabs(v);
        if (ms < av) ms = av;
    }
    mu = warp_max(mu);
    ms = warp_max(ms);
    if (bad) atomicAdd(&s_bad, bad);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) {
        s_u[w] = mu;
        s_s[w] = ms;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < static_cast<int>(blockDim.x / 32); ++q) {
            if (mu < s_u[q]) mu = s_u[q];
            if (ms < s_s[q]) ms = s_s[q];
        }
        atomicMax(&p.red[0], static_cast<unsigned long long>(__double_as_longlong(mu)));
        atomicMax(&p.red[1], static_cast<unsigned long long>(__double_as_longlong(ms)));
        if (s_bad) atomicAdd(&p.red[2], static_cast<unsigned long long>(s_bad));
    }
}

// End-of-step clipping (simulate.cpp:168-174): v < 0 -> 0, counted.
__global__ void __launch_bounds__(256) clip_kernel(int64_t n, double* y, unsigned long long* count) {
    unsigned int c = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (y[i] < 0.0) {
            y[i] = 0.0;
            ++c;
        }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, static_cast<unsigned long long>(c));
}

}  // namespace bc
