/*
 * bc_oracle.h -- CPU restatement of the reference Block-cells solver path.
 *
 * TEST INFRASTRUCTURE ONLY.  This oracle is the checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product library (libbc_b200.so) never links or calls it.
 *
 * Every function restates one reference function (file:line relative to
 * /root/reference/proj/core) with identical floating-point operation order,
 * so that, compiled with -ffp-contract=off on x86-64 (SSE2 doubles, no FMA),
 * it is bit-identical to the reference.  That claim is pinned by
 * tests/test_oracle.py against oracle/_ref (the reference compiled from its
 * own sources; for BICGSTAB_JACOBI, the same algorithm composed from the
 * reference's primitives, oracle/ref_bicgstab.cpp) and by the committed
 * golden fixtures in tests/golden/.
 *
 * BICGSTAB_JACOBI has no reference implementation: it is
 * defined here, using the reference's primitives (spmv, axpby-style updates,
 * the stride-halving tree reduction, RMS convergence with fresh-residual
 * confirmation, the 1e-300 breakdown floor).  It is pinned bitwise against
 * the same algorithm composed from the reference's compiled spmv / axpby /
 * plan_reduce_map / lu_solve and strategy drivers (oracle/ref_bicgstab.cpp),
 * and cross-checked against the reference's dense LU (lu_solve) on
 * converging systems.
 */
#ifndef BC_ORACLE_H
#define BC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_ERR_INVALID_ARGUMENT = -1,     /* std::invalid_argument            */
    ORC_ERR_INVALID_GROUPING = -2,     /* exec_model.hpp:19 InvalidGrouping */
    ORC_ERR_UNSUPPORTED_MECHANISM = -3,/* exec_model.hpp:14                 */
    ORC_ERR_SINGULAR_MATRIX = -4,      /* dense_lu.hpp:12 SingularMatrix    */
    ORC_ERR_NO_MEMORY = -7
};

enum { ORC_STRATEGY_ONE_CELL = 0, ORC_STRATEGY_MULTI_CELLS = 1, ORC_STRATEGY_BLOCK_CELLS = 2 };
enum { ORC_ALGO_BICG = 0, ORC_ALGO_BICGSTAB_JACOBI = 1 };

/* per-group flag bits */
enum { ORC_FLAG_CONVERGED = 1, ORC_FLAG_BREAKDOWN = 2, ORC_FLAG_FELL_BACK = 4 };

typedef struct {
    int64_t begin, end;
} orc_range;

typedef struct {
    int64_t iterations;
    double final_residual_rms;
    int32_t converged;
    int32_t breakdown;
} orc_outcome;

typedef struct {
    int64_t n_groups;
    int64_t iterations_effective;
    int64_t iterations_sum;
    double max_residual_rms;
    int64_t breakdown_fallbacks;
    double cells_per_block;
} orc_report;

/* reduction.cpp:38-44 */
double orc_tree_reduce_in_place(double* slots, int64_t padded_len);
/* reduction.hpp:60-79 over a precomputed value array; block_partials may be NULL */
double orc_plan_reduce(const double* values, int64_t n, const orc_range* ranges,
                       int64_t n_blocks, double* scratch, double* block_partials);

/* csr.cpp:90-101, 129-142, 150-156 (int64 CSR, as the reference's size_t) */
void orc_spmv(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx,
              const double* vals, const double* x, double* y);
void orc_spmv_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* vals, const double* x,
                        double* y);
void orc_axpby(int64_t n, double a, const double* x, double b, const double* y, double* z);

/* bicg.cpp:42-142; ranges = the ReductionPlan's block_ranges */
int orc_bicg_solve(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                   const double* vals, const double* b, const double* x0, double tol,
                   int64_t max_iter, const orc_range* ranges, int64_t n_blocks,
                   double* x_out, orc_outcome* out);
/* Jacobi-preconditioned BiCGSTAB, same conventions as above */
int orc_bicgstab_solve(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                       const double* vals, const double* b, const double* x0, double tol,
                       int64_t max_iter, const orc_range* ranges, int64_t n_blocks,
                       double* x_out, orc_outcome* out);

/* dense_lu.cpp:8-16 + 18-63 + 65-67 */
int orc_lu_solve_csr(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                     const double* vals, const double* b, double* x_out);

/* exec_model.cpp:102-161: the k the strategy will use (request 0 = "N" rule) */
int orc_plan_cells_per_block(int strategy, int64_t cells, int64_t species,
                             int64_t max_threads_per_block, int64_t k_request,
                             double* cells_per_block);

/*
 * strategies.cpp:158-264 (run_strategy) over a batch sharing one pattern.
 *   values: cells*nnz, cell-major, CSR order of the shared pattern
 *   rhs:    cells*species
 * Outputs: x_out cells*species; group_iters/group_rms/group_flags have
 * report->n_groups entries (callers size them with orc_group_count).
 */
int64_t orc_group_count(int strategy, int64_t cells, int64_t species,
                        int64_t max_threads_per_block, int64_t k_request);
int orc_solve_batch(int strategy, int algo, int64_t k_request, int64_t species,
                    int64_t cells, const int32_t* row_ptr, const int32_t* col_idx,
                    const double* values, const double* rhs, double tol,
                    int64_t max_iter, int64_t max_threads_per_block, int64_t workers,
                    double* x_out, int64_t* group_iters, double* group_rms,
                    uint8_t* group_flags, orc_report* report);

#ifdef __cplusplus
}
#endif
#endif
