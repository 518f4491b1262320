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

}  // namespace bc
