/*
 * blockcells_workload.h -- synthetic CB05-shaped workload (C ABI).
 *
 * Input synthesis for benchmarks and tests: the reference's synthetic
 * mechanism and the first backward-Euler Newton system of each cell,
 * restated so that values are bit-identical to the reference generator
 * (pinned by tests/test_workload.py against oracle/_ref):
 *   generate_mechanism     mechanism.cpp:117-150
 *   MechanismEvaluator     mechanism.cpp:172-219 (pattern + stamps)
 *   cell_conditions        mechanism.cpp:152-170
 *   rate_constants         mechanism.cpp:221-233
 *   rhs_into/jacobian_into mechanism.cpp:235-267
 *   fill_newton_system     simulate.cpp:29-42  (A = I - hJ, b = -(y - y_prev - h f))
 * The host fill is multi-threaded; bcw_newton_values_device (a CUDA kernel in
 * libbc_b200.so, blockcells_b200.h) assembles the same values on the GPU.
 */
#ifndef BLOCKCELLS_WORKLOAD_H
#define BLOCKCELLS_WORKLOAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bcw_mechanism bcw_mechanism;

enum { BCW_MODE_IDEAL = 0, BCW_MODE_REALISTIC = 1 };

/* generate_mechanism(species, reactions, seed) + its evaluator tables. */
int bcw_mechanism_create(int64_t species, int64_t reactions, uint64_t seed, bcw_mechanism** out);
/* Any mechanism (MechanismSpec, mechanism.hpp:30-40, as flat arrays: kind 0
 * emission / 1 unimolecular / 2 bimolecular, reactants and products in CSR
 * form) with the same evaluator tables. */
int bcw_mechanism_from_reactions(int64_t species, int64_t reactions, const int32_t* kind,
                                 const int32_t* reactant_ptr, const int32_t* reactants,
                                 const int32_t* product_ptr, const int32_t* products, const double* rate_coeff,
                                 const double* temp_exponent, bcw_mechanism** out);
void bcw_mechanism_destroy(bcw_mechanism* m);
int64_t bcw_species(const bcw_mechanism* m);
int64_t bcw_reactions(const bcw_mechanism* m);
int64_t bcw_nnz(const bcw_mechanism* m);
/* The shared Jacobian pattern (row_ptr: species+1, col_idx: nnz). */
int bcw_pattern(const bcw_mechanism* m, int32_t* row_ptr, int32_t* col_idx);

/*
 * Newton systems for cells [first, first+count) of a total_cells batch at
 * state y (cell-major, count*species; NULL = every species at 1.0) and
 * previous state y_prev (NULL = y).  values: count*nnz (CSR order of the
 * pattern), rhs: count*species.  threads <= 0 uses all hardware threads.
 */
int bcw_newton_batch(const bcw_mechanism* m, int64_t first, int64_t count, int64_t total_cells,
                     int mode, double h, const double* y, const double* y_prev, double* values,
                     double* rhs, int threads);

/*
 * Device-assembly tables (for the CUDA Newton-assembly kernel): per-cell
 * rate constants (count*reactions, host pow() as in rate_constants) and the
 * flattened stamp program.  See blockcells_b200.h bc_newton_assemble.
 */
int bcw_rate_constants(const bcw_mechanism* m, int64_t first, int64_t count,
                       int64_t total_cells, int mode, double* rates, int threads);
/* Stamp program: for reaction j, stamps [stamp_ptr[j], stamp_ptr[j+1]) with
 * slot, sign (+1/-1), other-reactant index (-1 when unimolecular), and the
 * reaction's reactant/product lists (CSR form, species indices). */
int64_t bcw_stamp_count(const bcw_mechanism* m);
int bcw_stamp_program(const bcw_mechanism* m, int32_t* stamp_ptr, int32_t* stamp_slot,
                      double* stamp_sign, int32_t* stamp_other, int32_t* reactant_ptr,
                      int32_t* reactants, int32_t* product_ptr, int32_t* products,
                      int32_t* diag_slot);

#ifdef __cplusplus
}
#endif
#endif
