/*
 * blockcells_b200.h -- C ABI of the B200-native Block-cells solver.
 *
 * This is the drop-in boundary for the reference's solver entry points in
 * /root/reference/proj/core (file:line below).  Plain pointers and sizes,
 * no C++ or torch types, no exceptions: a maintainer binds these from the
 * reference's C++ API with the shim in paper_2405_17363_b200/shim/
 * (see INTEGRATION.md).  Everything runs on the GPU (sm_100a); there is no
 * CPU solver path behind these entry points.
 *
 *   bc_solve        replaces run_strategy          strategies.hpp:80-82 (strategies.cpp:251-264)
 *                   i.e. solve_one_cell            strategies.hpp:60-61 (strategies.cpp:158-174)
 *                        solve_multi_cells         strategies.hpp:65-67 (strategies.cpp:176-194)
 *                        solve_block_cells         strategies.hpp:74-77 (strategies.cpp:196-249)
 *                   incl. the LU breakdown fallback strategies.cpp:37-69 / dense_lu.cpp:18-63
 *                   and merge_groups               strategies.cpp:71-87
 *   bc_bicg_solve   replaces bicg_solve            bicg.hpp:42-48 (bicg.cpp:42-142)
 *   bc_plan         mirrors plan_kernel's grouping exec_model.hpp:99-101 (exec_model.cpp:102-161)
 *
 * Error behaviour mirrors the reference's exceptions as status codes:
 *   BC_ERR_INVALID_ARGUMENT      std::invalid_argument (shape, pattern, tol<=0, max_iter<1)
 *   BC_ERR_INVALID_GROUPING      blockcells::InvalidGrouping      exec_model.hpp:19-21
 *   BC_ERR_UNSUPPORTED_MECHANISM blockcells::UnsupportedMechanism exec_model.hpp:14-16
 *   BC_ERR_SINGULAR_MATRIX       blockcells::SingularMatrix       dense_lu.hpp:12-14 (LU fallback)
 *   BC_ERR_SOLVER_ABORT          blockcells::SolverAbort          simulate.hpp:15-19 (bc_simulate)
 * Numerical breakdown is a per-group flag, never an error (bicg.hpp:39-41).
 *
 * Pointers passed to bc_solve / bc_bicg_solve may be host (pageable or
 * pinned) or device memory of the context's GPU; the library detects which.
 * Calls are synchronous with respect to the host (like the reference) but
 * run on the caller's stream.  A context is not thread-safe: use one per
 * calling thread (or guard it), one per GPU.
 */
#ifndef BLOCKCELLS_B200_H
#define BLOCKCELLS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BC_OK = 0,
    BC_ERR_INVALID_ARGUMENT = -1,
    BC_ERR_INVALID_GROUPING = -2,
    BC_ERR_UNSUPPORTED_MECHANISM = -3,
    BC_ERR_SINGULAR_MATRIX = -4,
    BC_ERR_CUDA = -5,
    BC_ERR_NO_PATTERN = -6,
    BC_ERR_NO_MEMORY = -7,
    BC_ERR_SOLVER_ABORT = -8
} bc_status;

/* Strategy (exec_model.hpp:23) plus the two comparison baselines. */
typedef enum {
    BC_STRATEGY_ONE_CELL = 0,        /* one cell per group, P = next_pow2(species)          */
    BC_STRATEGY_MULTI_CELLS = 1,     /* one global system, 1024-slot blocks + host stage    */
    BC_STRATEGY_BLOCK_CELLS = 2,     /* groups of k cells coupled in one Krylov solve        */
    BC_STRATEGY_THREAD_PER_CELL = 3  /* baseline: one thread solves one cell (= One-cell math) */
} bc_strategy;

typedef enum {
    BC_ALGO_BICG = 0,            /* the reference's two-sided BiCG (bicg.cpp), bit-exact */
    BC_ALGO_BICGSTAB_JACOBI = 1  /* Jacobi-preconditioned BiCGSTAB      */
} bc_algo;

/* per-group flag bits */
enum { BC_FLAG_CONVERGED = 1, BC_FLAG_BREAKDOWN = 2, BC_FLAG_FELL_BACK = 4 };

/* bc_solve_params.options */
enum {
    BC_OPT_TIMING = 1 /* fill bc_report.device_ms with CUDA-event time of the solver kernels */
};

typedef struct bc_ctx bc_ctx;

typedef struct {
    int32_t strategy;              /* bc_strategy                                          */
    int32_t algo;                  /* bc_algo                                              */
    int64_t cells_per_block;       /* Block-cells k; 0 = floor(max_threads_per_block/species) */
    int64_t cells;                 /* number of cells in values/rhs                         */
    double tol;                    /* RMS residual tolerance (> 0)                          */
    int64_t max_iter;              /* >= 1; iteration counts are int32: values above 2^31 - 2
                                      act as 2^31 - 2 (hours of iterations for one cell)     */
    int64_t max_threads_per_block; /* DeviceSpec::max_threads_per_block (0 = 1024)          */
    void* stream;                  /* cudaStream_t to run on (NULL = legacy default)        */
    int32_t options;               /* BC_OPT_*                                              */
    int32_t reserved;
} bc_solve_params;

/* SolveReport (strategies.hpp:35-48) minus per_cell_x / per_block_iterations
 * (returned through the x_out / group_iters arrays). */
typedef struct {
    int64_t n_groups;
    int64_t iterations_effective; /* max over groups */
    int64_t iterations_sum;       /* sum over groups */
    double max_residual_rms;
    int64_t breakdown_fallbacks;
    double cells_per_block;
    double device_ms;             /* solver kernels only, when BC_OPT_TIMING */
    int64_t kernel_launches;      /* kernels this call launched */
    int32_t kernels;              /* BC_KERNEL_* bits of the kernels this call launched */
    int32_t reserved;
    double model_spmv_wavefronts; /* TMEM kernel: the planner's modelled shared-memory wavefronts of
                                     one group-iteration's SpMVs (0 if it did not run) */
} bc_report;

enum {
    BC_KERNEL_TMEM = 1,   /* block_cells_tmem_kernel (both algorithms; one warp or a 2/4-warp team per group,
                             TMEM operands) */
    BC_KERNEL_BLOCK = 2,  /* block_cells_kernel (BiCG / wide groups, shared-memory operands) */
    BC_KERNEL_MULTI = 4,  /* multi_cells_kernel (cooperative, grid-wide reductions) */
    BC_KERNEL_THREAD = 8, /* thread_per_cell_kernel (+ interleave_kernel) */
    BC_KERNEL_LU = 16,    /* lu_fallback_kernel */
    BC_KERNEL_LATENCY = 32 /* block_cells_latency_kernel (small batches: one CTA, one thread per row) */
};

typedef struct {
    int64_t iterations;
    double final_residual_rms;
    int32_t converged;
    int32_t breakdown;
} bc_outcome; /* SolveOutcome (bicg.hpp:25-31) minus x */

/* Context bound to one CUDA device. */
int bc_ctx_create(int device, bc_ctx** out);
void bc_ctx_destroy(bc_ctx* ctx);
const char* bc_last_error(const bc_ctx* ctx);

/* The sparsity pattern shared by every cell (BatchedSystem::check,
 * strategies.cpp:91-107): species rows, CSR with strictly increasing
 * columns per row.  nnz = row_ptr[species].  Builds the device schedules. */
int bc_set_pattern(bc_ctx* ctx, int32_t species, const int32_t* row_ptr, const int32_t* col_idx);

/* The installed pattern's species and nnz (info[0], info[1]). */
int bc_ctx_pattern_info(const bc_ctx* ctx, int32_t* info);

/* Group geometry of a solve (plan_kernel + solve_block_cells partition):
 * number of groups and the k used (fractional for Multi-cells). */
int bc_plan(int32_t species, const bc_solve_params* prm, int64_t* n_groups,
            double* cells_per_block);

/* Host-side schedule of the fused kernel for a pattern and group size k
 * (no GPU needed; for tests and DESIGN.md).  info[0..11] = n, P, Q, W, R,
 * RV, S (A steps), St (A^T steps, 0 unless with_transpose), xslots,
 * txslots (shared slots of the gathered vectors), modelled gather
 * wavefronts of one A pass and one A^T pass.  The array outputs may be NULL
 * to query sizes: words S*W*32, vpos k*nnz, xpos n (row -> gather slot). */
int bc_schedule_export(int32_t species, const int32_t* row_ptr, const int32_t* col_idx, int32_t k,
                       int32_t with_transpose, int32_t* info, uint32_t* words, int32_t* vpos,
                       int32_t* xpos, uint32_t* twords, int32_t* tvpos, int32_t* txpos);

/* Schedule of the Tensor-Memory kernel (one warp per group; see
 * paper_2405_17363_b200/csrc/bc_plan.hpp TmemSchedule).  info[0..8] = S
 * (steps, multiple of 4), xslots, zero_slot, yslots, modelled gather
 * wavefronts per pass, copies of the gather vector, modelled shared
 * wavefronts per SpMV, row streams per lane, Y slots per stream.  pair != 0:
 * BiCG's schedule, A rows on stream 0 and A^T rows on stream 1 (columns and
 * outputs doubled).  team: warps per group (1, 2, 4).  Arrays may be NULL to
 * query sizes: words/vidx S*32*team, xpos copies*k*species (x2 for a pair),
 * yslot k*species (x2 for a pair). */
int bc_tmem_schedule_export(int32_t species, const int32_t* row_ptr, const int32_t* col_idx, int32_t k,
                            int32_t pair, int32_t team, int32_t* info, uint16_t* words, int32_t* vidx,
                            int32_t* xpos, int32_t* yslot);

/* Schedule of the latency-mode kernel (csrc/bc_latency.cuh; bc_plan.hpp
 * LatencySchedule) for a group of k cells and a kernel instance of `threads`
 * threads (no GPU needed; for tests).  info[0..7] = n, P, T (threads), lmax
 * (longest row, A^T row too for bicg), L (padded steps: the [L][T] tables),
 * xslots (doubles of one warp's gather region), modelled gather wavefronts
 * of one SpMV, 1 if tables were produced (lmax <= 32).  Arrays (NULL to skip):
 * rowof/steps [T], rvi/rxo (and for bicg tvi/txo) [L][T], didx [P]. */
int bc_latency_schedule_export(int32_t species, const int32_t* row_ptr, const int32_t* col_idx, int32_t k,
                               int32_t bicg, int32_t threads, int32_t* info, int32_t* rowof, int32_t* steps,
                               int32_t* rvi, uint16_t* rxo, int32_t* tvi, uint16_t* txo, int32_t* didx);

/*
 * Solve every cell's system A_c x_c = b_c (x0 = 0, as solve_group does).
 *   values: cells * nnz fp64, cell-major, each cell in the pattern's CSR order
 *           (= BatchedSystem::per_cell_matrices[c].values back to back)
 *   rhs:    cells * species fp64 (= per_cell_rhs back to back)
 *   x_out:  cells * species fp64 (= SolveReport::per_cell_x back to back)
 *   group_iters / group_rms / group_flags: n_groups entries each, or NULL
 *   report: may be NULL
 */
int bc_solve(bc_ctx* ctx, const bc_solve_params* prm, const double* values, const double* rhs,
             double* x_out, int32_t* group_iters, double* group_rms, uint8_t* group_flags,
             bc_report* report);

/*
 * One system with its own pattern (bicg_solve, bicg.hpp:42-48).  The
 * ReductionPlan is given as n_blocks [begin,end) pairs partitioning [0,n);
 * x0 may be NULL (zeros).  algo selects BiCG or Jacobi-BiCGSTAB.
 */
int bc_bicg_solve(bc_ctx* ctx, int32_t algo, int32_t n, const int32_t* row_ptr,
                  const int32_t* col_idx, const double* vals, const double* b, const double* x0,
                  double tol, int64_t max_iter, int64_t n_blocks, const int64_t* ranges,
                  double* x_out, bc_outcome* out);

/* Number of kernels launched since context creation (evidence counter). */
int64_t bc_kernel_launches(const bc_ctx* ctx);

/*
 * Device set: the drop-in API over several GPUs of one box,
 * the GPU counterpart of solve_block_cells' worker pool
 * (strategies.cpp:221-247).  One bc_ctx and one stream per device (a device
 * may be listed twice: two contexts on one GPU).  bc_devset_solve shards the
 * batch into contiguous group-aligned cell ranges (the leftover group on the
 * last shard), runs one host thread per device, and merges the report in
 * group order as merge_groups (strategies.cpp:71-87) does: every output is
 * bit-identical to bc_solve on one device.  No collective.  Multi-cells runs
 * on the first device only (one global system).  With more than one device
 * the arrays must be host memory (pageable or pinned).
 */
typedef struct bc_devset bc_devset;
/* Pinned, portable, mapped host staging memory (cudaHostAlloc), for callers
 * that pack into it: host inputs in pinned memory stream into the solve
 * while it runs, and a pinned x_out is written by the kernels in place. */
int bc_host_alloc(uint64_t bytes, void** out);
void bc_host_free(void* p);

int bc_devset_create(int n_devices, const int* devices, bc_devset** out);
void bc_devset_destroy(bc_devset* set);
int bc_devset_size(const bc_devset* set);
const char* bc_devset_last_error(const bc_devset* set);
int bc_devset_set_pattern(bc_devset* set, int32_t species, const int32_t* row_ptr, const int32_t* col_idx);
int bc_devset_solve(bc_devset* set, const bc_solve_params* prm, const double* values, const double* rhs,
                    double* x_out, int32_t* group_iters, double* group_rms, uint8_t* group_flags,
                    bc_report* report);

/*
 * Device Newton-system assembly (simulate.cpp:29-42 +
 * mechanism.cpp:235-267).  From per-cell rate constants (host pow(), see
 * blockcells_workload.h bcw_rate_constants) and the mechanism's stamp
 * program, writes values (count*nnz) and rhs (count*species) for states
 * y / y_prev (count*species each; NULL = all ones / = y).  Bit-identical to
 * bcw_newton_batch.  Pointers: device memory.
 */
int bc_newton_assemble(bc_ctx* ctx, int64_t count, int32_t species, int32_t reactions,
                       int32_t nnz, const double* rates, const int32_t* stamp_ptr,
                       const int32_t* stamp_slot, const double* stamp_sign,
                       const int32_t* stamp_other, const int32_t* reactant_ptr,
                       const int32_t* reactants, const int32_t* product_ptr,
                       const int32_t* products, const int32_t* diag_slot, double h,
                       const double* y, const double* y_prev, double* values, double* rhs,
                       void* stream);

/*
 * Device-resident backward-Euler simulation: replaces
 * run_simulation (simulate.hpp:76-78, simulate.cpp:72-178) with every
 * per-cell array kept in HBM.  Per Newton iteration: bc_newton_assemble's
 * kernel builds A = I - hJ(y), b = -(y - y_prev - h f(y)) from the current
 * states; the configured strategy solves (bc_solve on device memory), or the
 * device LU when use_direct_reference; one fused kernel adds the update and
 * max-reduces |dy| and |y| (max is order-free, so bit-equal to the host
 * loop); only those two numbers cross to the host for the Newton test
 * |dy|_inf < newton_rtol * |y|_inf.  Negative states are clipped (counted)
 * after each step.  A non-finite state returns BC_ERR_SOLVER_ABORT with
 * *abort_step set, as SolverAbort does.
 */
typedef struct { /* SimulationConfig (simulate.hpp:39-55) */
    int64_t cells;
    int64_t steps;
    double dt_seconds;
    double tol;
    int64_t max_iter;
    int32_t strategy;             /* bc_strategy                          */
    int32_t algo;                 /* bc_algo                              */
    int64_t cells_per_block;      /* 0 = "N"                              */
    int64_t max_threads_per_block;
    int32_t use_direct_reference; /* LinearSolverChoice: dense LU per cell */
    int32_t reserved;
    double newton_rtol;
    int64_t max_newton_iterations;
    void* stream;
} bc_sim_params;

typedef struct { /* StepStats (simulate.hpp:59-68) */
    int64_t step;
    int64_t newton_iterations;
    int64_t iterations_effective;
    int64_t iterations_sum;
    double max_residual_rms;
    int64_t wall_time_ns;
    int64_t breakdown_fallbacks;
    int64_t clip_events;
} bc_step_stats;

typedef struct { /* the mechanism's evaluator tables (blockcells_workload.h bcw_stamp_program), host memory */
    int32_t species, reactions, nnz, stamps;
    const int32_t *row_ptr, *col_idx; /* Jacobian pattern */
    const int32_t *stamp_ptr, *stamp_slot, *stamp_other;
    const double* stamp_sign;
    const int32_t *reactant_ptr, *reactants, *product_ptr, *products, *diag_slot;
} bc_mechanism_tables;

/* rates: cells*reactions (host, rate_constants per cell); states: cells*species
 * (host or device) in: initial states, out: final states; per_step: steps
 * entries (host). */
int bc_simulate(bc_ctx* ctx, const bc_sim_params* prm, const bc_mechanism_tables* mech,
                const double* rates, double* states, bc_step_stats* per_step, int64_t* abort_step);

#ifdef __cplusplus
}
#endif
#endif
