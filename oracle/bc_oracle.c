/*
 * bc_oracle.c -- CPU restatement of the reference Block-cells solver path.
 * TEST INFRASTRUCTURE ONLY (see bc_oracle.h).  Compile with
 * -ffp-contract=off and without -ffast-math / -march (no FMA contraction).
 *
 * Citations are relative to /root/reference/proj/core.
 */
#include "bc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ORC_BREAKDOWN_FLOOR 1e-300 /* bicg.cpp:10 kBreakdownFloor */

/* bicg.cpp:12-14 scalar_breaks */
static int scalar_breaks(double v) { return !isfinite(v) || fabs(v) < ORC_BREAKDOWN_FLOOR; }

/* reduction.cpp:34-36 detail::padded_block_len (bit_ceil, 1 for n<=1) */
static int64_t padded_block_len(int64_t n) {
    if (n <= 1) return 1;
    int64_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

/* reduction.cpp:38-44 tree_reduce_in_place: stride-halving pairwise tree */
double orc_tree_reduce_in_place(double* slots, int64_t padded_len) {
    for (int64_t stride = padded_len / 2; stride >= 1; stride /= 2)
        for (int64_t i = 0; i < stride; ++i) slots[i] += slots[i + stride];
    return slots[0];
}

/* reduction.hpp:60-79 plan_reduce_map: per-interval tree, then the
 * sequential left-to-right combine of the block partials. */
double orc_plan_reduce(const double* values, int64_t n, const orc_range* ranges,
                       int64_t n_blocks, double* scratch, double* block_partials) {
    (void)n;
    double total = 0.0;
    for (int64_t b = 0; b < n_blocks; ++b) {
        const int64_t len = ranges[b].end - ranges[b].begin;
        const int64_t padded = padded_block_len(len);
        for (int64_t i = 0; i < padded; ++i) scratch[i] = 0.0;
        for (int64_t i = 0; i < len; ++i) scratch[i] = values[ranges[b].begin + i];
        const double partial = orc_tree_reduce_in_place(scratch, padded);
        if (block_partials) block_partials[b] = partial;
        total = (b == 0) ? partial : total + partial;
    }
    return total;
}

/* reduction.cpp:16-25 check_partition */
static int check_partition(const orc_range* ranges, int64_t n_blocks, int64_t n) {
    int64_t expect = 0;
    for (int64_t b = 0; b < n_blocks; ++b) {
        if (ranges[b].begin != expect || ranges[b].end <= ranges[b].begin) return 0;
        expect = ranges[b].end;
    }
    return expect == n;
}

/* csr.cpp:90-101 spmv: each row accumulated from 0.0 in storage order */
void orc_spmv(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx,
              const double* vals, const double* x, double* y) {
    for (int64_t i = 0; i < n_rows; ++i) {
        double sum = 0.0;
        const int64_t end = row_ptr[i + 1];
        for (int64_t j = row_ptr[i]; j < end; ++j) sum += vals[j] * x[col_idx[j]];
        y[i] = sum;
    }
}

/* csr.cpp:129-142 spmv_transpose: scatter in ascending row order */
void orc_spmv_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* vals, const double* x,
                        double* y) {
    for (int64_t j = 0; j < n_cols; ++j) y[j] = 0.0;
    for (int64_t i = 0; i < n_rows; ++i) {
        const double xi = x[i];
        for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) y[col_idx[j]] += vals[j] * xi;
    }
}

/* csr.cpp:150-156 axpby: z = a*x + b*y (two products, then the add) */
void orc_axpby(int64_t n, double a, const double* x, double b, const double* y, double* z) {
    for (int64_t i = 0; i < n; ++i) z[i] = a * x[i] + b * y[i];
}

/* ------------------------------------------------------------------ */
/* Reduction helpers over the plan (value arrays are formed on the fly  */
/* exactly as plan_reduce_map's lambdas do).                            */

typedef struct {
    const orc_range* ranges;
    int64_t n_blocks;
    double* scratch; /* >= max padded block length */
    double* vals;    /* n temporaries */
} orc_plan_ctx;

static double reduce_prod(orc_plan_ctx* pc, int64_t n, const double* a, const double* b) {
    for (int64_t i = 0; i < n; ++i) pc->vals[i] = a[i] * b[i];
    return orc_plan_reduce(pc->vals, n, pc->ranges, pc->n_blocks, pc->scratch, NULL);
}

/* bicg.cpp:61-72 residual_rms: sqrt(plan_reduce((b-Ax)^2)/n) */
static double residual_rms(orc_plan_ctx* pc, int64_t n, const int64_t* rp, const int64_t* ci,
                           const double* va, const double* b, const double* x, double* ax) {
    orc_spmv(n, rp, ci, va, x, ax);
    for (int64_t i = 0; i < n; ++i) {
        const double ri = b[i] - ax[i];
        pc->vals[i] = ri * ri;
    }
    const double sq = orc_plan_reduce(pc->vals, n, pc->ranges, pc->n_blocks, pc->scratch, NULL);
    return sqrt(sq / (double)n);
}

static int64_t max_padded(const orc_range* ranges, int64_t n_blocks) {
    int64_t m = 1;
    for (int64_t b = 0; b < n_blocks; ++b) {
        const int64_t p = padded_block_len(ranges[b].end - ranges[b].begin);
        if (p > m) m = p;
    }
    return m;
}

/* bicg.cpp:42-142 bicg_solve (unpreconditioned two-sided BiCG) */
int orc_bicg_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                   const double* b, const double* x0, double tol, int64_t max_iter,
                   const orc_range* ranges, int64_t n_blocks, double* x, orc_outcome* out) {
    if (!(tol > 0.0)) return ORC_ERR_INVALID_ARGUMENT;
    if (max_iter < 1) return ORC_ERR_INVALID_ARGUMENT;
    if (!check_partition(ranges, n_blocks, n)) return ORC_ERR_INVALID_ARGUMENT;

    double* buf = (double*)malloc(sizeof(double) * (size_t)(8 * n + max_padded(ranges, n_blocks)));
    if (!buf) return ORC_ERR_NO_MEMORY;
    double *r = buf, *rs = buf + n, *p = buf + 2 * n, *ps = buf + 3 * n, *ap = buf + 4 * n,
           *atps = buf + 5 * n, *vals = buf + 6 * n, *scratch = buf + 8 * n;
    orc_plan_ctx pc = {ranges, n_blocks, scratch, vals};

    memset(out, 0, sizeof *out);
    memcpy(x, x0, sizeof(double) * (size_t)n);

    orc_spmv(n, rp, ci, va, x, ap);                 /* bicg.cpp:74 */
    orc_axpby(n, 1.0, b, -1.0, ap, r);              /* bicg.cpp:75 */
    memcpy(rs, r, sizeof(double) * (size_t)n);      /* bicg.cpp:76-78 */
    memcpy(p, r, sizeof(double) * (size_t)n);
    memcpy(ps, rs, sizeof(double) * (size_t)n);

    double rho_prev = 0.0;
    double recurrence_sq = reduce_prod(&pc, n, r, r); /* bicg.cpp:81-83 */
    if (sqrt(recurrence_sq / (double)n) <= tol) {      /* bicg.cpp:87-91 */
        out->final_residual_rms = residual_rms(&pc, n, rp, ci, va, b, x, ap);
        out->converged = out->final_residual_rms <= tol;
        if (out->converged) { free(buf); return ORC_OK; }
    }

    for (int64_t iter = 1; iter <= max_iter; ++iter) {  /* bicg.cpp:93-137 */
        const double rho = reduce_prod(&pc, n, rs, r);
        if (scalar_breaks(rho)) { out->breakdown = 1; break; }
        if (iter > 1) {
            const double beta = rho / rho_prev;
            orc_axpby(n, 1.0, r, beta, p, p);
            orc_axpby(n, 1.0, rs, beta, ps, ps);
        }
        orc_spmv(n, rp, ci, va, p, ap);
        orc_spmv_transpose(n, n, rp, ci, va, ps, atps);
        const double denom = reduce_prod(&pc, n, ps, ap);
        if (scalar_breaks(denom)) { out->breakdown = 1; break; }
        const double alpha = rho / denom;
        orc_axpby(n, 1.0, x, alpha, p, x);
        orc_axpby(n, 1.0, r, -alpha, ap, r);
        orc_axpby(n, 1.0, rs, -alpha, atps, rs);
        rho_prev = rho;
        out->iterations = iter;

        recurrence_sq = reduce_prod(&pc, n, r, r);
        if (!isfinite(recurrence_sq)) { out->breakdown = 1; break; }
        if (sqrt(recurrence_sq / (double)n) <= tol) {
            const double fresh = residual_rms(&pc, n, rp, ci, va, b, x, ap);
            if (fresh <= tol) {
                out->final_residual_rms = fresh;
                out->converged = 1;
                free(buf);
                return ORC_OK;
            }
        }
    }
    out->final_residual_rms = residual_rms(&pc, n, rp, ci, va, b, x, ap); /* bicg.cpp:139-141 */
    out->converged = !out->breakdown && out->final_residual_rms <= tol;
    free(buf);
    return ORC_OK;
}

/*
 * Jacobi-preconditioned BiCGSTAB (no reference code).
 * Pinned semantics, mirrored operation-for-operation by the CUDA kernel:
 *   dinv_i = 1.0 / a_ii   (a_ii the stored diagonal; 1.0 if absent or zero)
 *   setup as bicg.cpp:74-91: x=x0, r = 1*b + (-1)*A x, rh = r, p = v = 0,
 *         rho_prev = alpha = omega = 1, zero-iteration convergence check.
 *   iteration:
 *     rho = <rh,r>                         breakdown if scalar_breaks
 *     beta = (rho/rho_prev) * (alpha/omega)
 *     p_i = r_i + beta*(p_i - omega*v_i);  y_i = dinv_i*p_i;  v = A y
 *     den = <rh,v>                         breakdown if scalar_breaks
 *     alpha = rho/den
 *     s_i = r_i - alpha*v_i;  z_i = dinv_i*s_i;  x_i = x_i + alpha*y_i
 *     t = A z;  tt = <t,t>;  ts = <t,s>    breakdown if tt != 0 && scalar_breaks(tt)
 *     omega = tt == 0 ? 0 : ts/tt          (t = 0: s vanished, finish below)
 *     x_i = x_i + omega*z_i;  r_i = s_i - omega*t_i
 *     rho_prev = rho; iterations = iter
 *     sigma = <r,r>                        breakdown if !isfinite
 *     rms(sigma) <= tol and fresh rms <= tol  => converged
 *     scalar_breaks(omega)                 => breakdown
 *   exit as bicg.cpp:139-141 (fresh residual always reported).
 * Every <.,.> is plan_reduce over the element products, as in bicg.cpp.
 */
int orc_bicgstab_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                       const double* b, const double* x0, double tol, int64_t max_iter,
                       const orc_range* ranges, int64_t n_blocks, double* x, orc_outcome* out) {
    if (!(tol > 0.0)) return ORC_ERR_INVALID_ARGUMENT;
    if (max_iter < 1) return ORC_ERR_INVALID_ARGUMENT;
    if (!check_partition(ranges, n_blocks, n)) return ORC_ERR_INVALID_ARGUMENT;

    double* buf = (double*)malloc(sizeof(double) * (size_t)(12 * n + max_padded(ranges, n_blocks)));
    if (!buf) return ORC_ERR_NO_MEMORY;
    double *r = buf, *rh = buf + n, *p = buf + 2 * n, *v = buf + 3 * n, *y = buf + 4 * n,
           *s = buf + 5 * n, *z = buf + 6 * n, *t = buf + 7 * n, *dinv = buf + 8 * n,
           *ax = buf + 9 * n, *vals = buf + 10 * n, *scratch = buf + 12 * n;
    orc_plan_ctx pc = {ranges, n_blocks, scratch, vals};

    memset(out, 0, sizeof *out);
    memcpy(x, x0, sizeof(double) * (size_t)n);

    for (int64_t i = 0; i < n; ++i) {
        double d = 0.0;
        for (int64_t j = rp[i]; j < rp[i + 1]; ++j)
            if (ci[j] == i) { d = va[j]; break; }
        dinv[i] = (d != 0.0) ? 1.0 / d : 1.0;
    }

    orc_spmv(n, rp, ci, va, x, ax);
    orc_axpby(n, 1.0, b, -1.0, ax, r);
    memcpy(rh, r, sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) { p[i] = 0.0; v[i] = 0.0; }

    double sigma = reduce_prod(&pc, n, r, r);
    if (sqrt(sigma / (double)n) <= tol) {
        out->final_residual_rms = residual_rms(&pc, n, rp, ci, va, b, x, ax);
        out->converged = out->final_residual_rms <= tol;
        if (out->converged) { free(buf); return ORC_OK; }
    }

    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    for (int64_t iter = 1; iter <= max_iter; ++iter) {
        const double rho = reduce_prod(&pc, n, rh, r);
        if (scalar_breaks(rho)) { out->breakdown = 1; break; }
        const double beta = (rho / rho_prev) * (alpha / omega);
        for (int64_t i = 0; i < n; ++i) {
            p[i] = r[i] + beta * (p[i] - omega * v[i]);
            y[i] = dinv[i] * p[i];
        }
        orc_spmv(n, rp, ci, va, y, v);
        const double den = reduce_prod(&pc, n, rh, v);
        if (scalar_breaks(den)) { out->breakdown = 1; break; }
        alpha = rho / den;
        for (int64_t i = 0; i < n; ++i) {
            s[i] = r[i] - alpha * v[i];
            z[i] = dinv[i] * s[i];
            x[i] = x[i] + alpha * y[i];
        }
        orc_spmv(n, rp, ci, va, z, t);
        const double tt = reduce_prod(&pc, n, t, t);
        const double ts = reduce_prod(&pc, n, t, s);
        /* tt == 0 exactly: t = 0, i.e. s already vanished; omega = 0 lets the
         * convergence test below finish the solve (x = x + alpha*y). */
        if (tt != 0.0 && scalar_breaks(tt)) { out->breakdown = 1; break; }
        omega = tt == 0.0 ? 0.0 : ts / tt;
        for (int64_t i = 0; i < n; ++i) {
            x[i] = x[i] + omega * z[i];
            r[i] = s[i] - omega * t[i];
        }
        rho_prev = rho;
        out->iterations = iter;

        sigma = reduce_prod(&pc, n, r, r);
        if (!isfinite(sigma)) { out->breakdown = 1; break; }
        if (sqrt(sigma / (double)n) <= tol) {
            const double fresh = residual_rms(&pc, n, rp, ci, va, b, x, ax);
            if (fresh <= tol) {
                out->final_residual_rms = fresh;
                out->converged = 1;
                free(buf);
                return ORC_OK;
            }
        }
        if (scalar_breaks(omega)) { out->breakdown = 1; break; }
    }
    out->final_residual_rms = residual_rms(&pc, n, rp, ci, va, b, x, ax);
    out->converged = !out->breakdown && out->final_residual_rms <= tol;
    free(buf);
    return ORC_OK;
}

/* dense_lu.cpp:8-16 densify + 18-63 lu_solve: partial pivoting, max
 * magnitude with ties to the lowest row, row permutation via perm[]. */
int orc_lu_solve_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                     const double* b, double* x) {
    double* lu = (double*)calloc((size_t)(n * n), sizeof(double));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    if (!lu || !perm) { free(lu); free(perm); return ORC_ERR_NO_MEMORY; }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = rp[i]; j < rp[i + 1]; ++j) lu[i * n + ci[j]] = va[j];
    for (int64_t i = 0; i < n; ++i) perm[i] = i;

    for (int64_t k = 0; k < n; ++k) {
        int64_t pivot = k;
        double best = fabs(lu[perm[k] * n + k]);
        for (int64_t i = k + 1; i < n; ++i) {
            const double mag = fabs(lu[perm[i] * n + k]);
            if (mag > best) { best = mag; pivot = i; }
        }
        if (best == 0.0) { free(lu); free(perm); return ORC_ERR_SINGULAR_MATRIX; }
        const int64_t tmp = perm[k]; perm[k] = perm[pivot]; perm[pivot] = tmp;
        const double pivot_value = lu[perm[k] * n + k];
        for (int64_t i = k + 1; i < n; ++i) {
            double* lik = &lu[perm[i] * n + k];
            *lik /= pivot_value;
            const double factor = *lik;
            for (int64_t j = k + 1; j < n; ++j)
                lu[perm[i] * n + j] -= factor * lu[perm[k] * n + j];
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        double sum = b[perm[i]];
        for (int64_t j = 0; j < i; ++j) sum -= lu[perm[i] * n + j] * x[j];
        x[i] = sum;
    }
    for (int64_t ii = n; ii-- > 0;) {
        double sum = x[ii];
        for (int64_t j = ii + 1; j < n; ++j) sum -= lu[perm[ii] * n + j] * x[j];
        x[ii] = sum / lu[perm[ii] * n + ii];
    }
    free(lu);
    free(perm);
    return ORC_OK;
}

/* exec_model.cpp:102-161 plan_kernel, only the parts that fix semantics */
int orc_plan_cells_per_block(int strategy, int64_t cells, int64_t species, int64_t mtpb,
                             int64_t k_request, double* cpb) {
    if (mtpb <= 0) return ORC_ERR_INVALID_ARGUMENT;
    if (cells < 1 || species < 1) return ORC_ERR_INVALID_ARGUMENT;
    if (species > mtpb) return ORC_ERR_UNSUPPORTED_MECHANISM;
    switch (strategy) {
        case ORC_STRATEGY_ONE_CELL: *cpb = 1.0; return ORC_OK;
        case ORC_STRATEGY_MULTI_CELLS: *cpb = (double)mtpb / (double)species; return ORC_OK;
        case ORC_STRATEGY_BLOCK_CELLS: {
            int64_t k;
            if (k_request > 0) {
                k = k_request;
                if (k * species > mtpb) return ORC_ERR_INVALID_GROUPING;
            } else if (k_request == 0) {
                k = mtpb / species;
            } else {
                return ORC_ERR_INVALID_ARGUMENT;
            }
            *cpb = (double)k;
            return ORC_OK;
        }
    }
    return ORC_ERR_INVALID_ARGUMENT;
}

int64_t orc_group_count(int strategy, int64_t cells, int64_t species, int64_t mtpb,
                        int64_t k_request) {
    double cpb = 0.0;
    if (orc_plan_cells_per_block(strategy, cells, species, mtpb, k_request, &cpb) != ORC_OK)
        return -1;
    if (strategy == ORC_STRATEGY_ONE_CELL) return cells;
    if (strategy == ORC_STRATEGY_MULTI_CELLS) return 1;
    const int64_t k = (int64_t)cpb;
    return cells / k + (cells % k ? 1 : 0);
}

/* ------------------------------------------------------------------ */
/* strategies.cpp: groups, solve_group, merge_groups                    */

typedef struct {
    int algo;
    int64_t species, nnz;
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const double* values;
    const double* rhs;
    double tol;
    int64_t max_iter;
    double* x_out;
    /* groups */
    int64_t n_groups;
    const int64_t* g_begin; /* cell range per group */
    const int64_t* g_end;
    int64_t block_width; /* reduction interval width (multi-cells); 0 = single interval */
    int64_t* g_iters;
    double* g_rms;
    uint8_t* g_flags;
    /* scheduling */
    int64_t next;
    pthread_mutex_t lock;
    int status;
} orc_batch_job;

/* strategies.cpp:121-156 assemble_block_diagonal + 37-69 solve_group */
static int solve_group(orc_batch_job* job, int64_t g) {
    const int64_t c0 = job->g_begin[g], c1 = job->g_end[g];
    const int64_t s = job->species, nnz = job->nnz, cells = c1 - c0, n = cells * s;
    int64_t* rp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t* ci = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cells * nnz));
    double* b = (double*)malloc(sizeof(double) * (size_t)n);
    double* x0 = (double*)calloc((size_t)n, sizeof(double));
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t n_blocks = 1;
    if (job->block_width > 0) n_blocks = (n + job->block_width - 1) / job->block_width;
    orc_range* ranges = (orc_range*)malloc(sizeof(orc_range) * (size_t)n_blocks);
    int st = ORC_OK;
    if (!rp || !ci || !b || !x0 || !x || !ranges) { st = ORC_ERR_NO_MEMORY; goto done; }

    rp[0] = 0;
    for (int64_t c = 0; c < cells; ++c) {
        const int64_t shift = c * s;
        for (int64_t i = 0; i < s; ++i) {
            for (int64_t j = job->row_ptr[i]; j < job->row_ptr[i + 1]; ++j)
                ci[c * nnz + j] = job->col_idx[j] + shift;
            rp[c * s + i + 1] = c * nnz + job->row_ptr[i + 1];
        }
        memcpy(b + c * s, job->rhs + (c0 + c) * s, sizeof(double) * (size_t)s);
    }
    const double* va = job->values + c0 * nnz;
    if (job->block_width > 0) { /* exec_model.cpp:202-220 */
        for (int64_t k = 0; k < n_blocks; ++k) {
            ranges[k].begin = k * job->block_width;
            ranges[k].end = (k + 1) * job->block_width < n ? (k + 1) * job->block_width : n;
        }
    } else {
        ranges[0].begin = 0;
        ranges[0].end = n;
    }

    orc_outcome out;
    st = job->algo == ORC_ALGO_BICG
             ? orc_bicg_solve(n, rp, ci, va, b, x0, job->tol, job->max_iter, ranges, n_blocks, x, &out)
             : orc_bicgstab_solve(n, rp, ci, va, b, x0, job->tol, job->max_iter, ranges, n_blocks, x, &out);
    if (st != ORC_OK) goto done;
    uint8_t flags = (uint8_t)((out.converged ? ORC_FLAG_CONVERGED : 0) |
                              (out.breakdown ? ORC_FLAG_BREAKDOWN : 0));
    double rms = out.final_residual_rms;
    if (out.breakdown) { /* strategies.cpp:46-60 */
        st = orc_lu_solve_csr(n, rp, ci, va, b, x);
        if (st != ORC_OK) goto done;
        flags |= ORC_FLAG_FELL_BACK;
        double* ax = x0; /* reuse */
        double* vals = (double*)malloc(sizeof(double) * (size_t)n);
        double* scratch = (double*)malloc(sizeof(double) * (size_t)max_padded(ranges, n_blocks));
        if (!vals || !scratch) { free(vals); free(scratch); st = ORC_ERR_NO_MEMORY; goto done; }
        orc_spmv(n, rp, ci, va, x, ax);
        for (int64_t i = 0; i < n; ++i) {
            const double ri = b[i] - ax[i];
            vals[i] = ri * ri;
        }
        const double sq = orc_plan_reduce(vals, n, ranges, n_blocks, scratch, NULL);
        rms = sqrt(sq / (double)n);
        free(vals);
        free(scratch);
    }
    memcpy(job->x_out + c0 * s, x, sizeof(double) * (size_t)n);
    job->g_iters[g] = out.iterations;
    job->g_rms[g] = rms;
    job->g_flags[g] = flags;
done:
    free(rp); free(ci); free(b); free(x0); free(x); free(ranges);
    return st;
}

static void* batch_worker(void* arg) {
    orc_batch_job* job = (orc_batch_job*)arg;
    for (;;) {
        pthread_mutex_lock(&job->lock);
        const int64_t g = job->next++;
        const int failed = job->status != ORC_OK;
        pthread_mutex_unlock(&job->lock);
        if (g >= job->n_groups || failed) return NULL;
        const int st = solve_group(job, g);
        if (st != ORC_OK) {
            pthread_mutex_lock(&job->lock);
            if (job->status == ORC_OK) job->status = st;
            pthread_mutex_unlock(&job->lock);
        }
    }
}

/* strategies.cpp:251-264 run_strategy -> solve_one_cell / solve_multi_cells /
 * solve_block_cells, then merge_groups (strategies.cpp:71-87). */
int orc_solve_batch(int strategy, int algo, int64_t k_request, int64_t species, int64_t cells,
                    const int32_t* row_ptr, const int32_t* col_idx, const double* values,
                    const double* rhs, double tol, int64_t max_iter, int64_t mtpb,
                    int64_t workers, double* x_out, int64_t* group_iters, double* group_rms,
                    uint8_t* group_flags, orc_report* report) {
    if (cells < 1 || species < 1) return ORC_ERR_INVALID_ARGUMENT; /* strategies.cpp:92-95 */
    if (algo != ORC_ALGO_BICG && algo != ORC_ALGO_BICGSTAB_JACOBI) return ORC_ERR_INVALID_ARGUMENT;
    double cpb = 0.0;
    int st = orc_plan_cells_per_block(strategy, cells, species, mtpb, k_request, &cpb);
    if (st != ORC_OK) return st;
    if (!(tol > 0.0) || max_iter < 1) return ORC_ERR_INVALID_ARGUMENT;

    const int64_t n_groups = orc_group_count(strategy, cells, species, mtpb, k_request);
    int64_t* gb = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_groups);
    int64_t* ge = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_groups);
    if (!gb || !ge) { free(gb); free(ge); return ORC_ERR_NO_MEMORY; }
    int64_t block_width = 0;
    if (strategy == ORC_STRATEGY_ONE_CELL) {
        for (int64_t c = 0; c < cells; ++c) { gb[c] = c; ge[c] = c + 1; }
    } else if (strategy == ORC_STRATEGY_MULTI_CELLS) {
        gb[0] = 0; ge[0] = cells;
        block_width = mtpb;
    } else { /* strategies.cpp:209-213: full groups of k, then the leftover */
        const int64_t k = (int64_t)cpb;
        int64_t g = 0;
        for (int64_t c = 0; c + k <= cells; c += k, ++g) { gb[g] = c; ge[g] = c + k; }
        if (cells % k) { gb[g] = cells - cells % k; ge[g] = cells; }
    }

    orc_batch_job job;
    memset(&job, 0, sizeof job);
    job.algo = algo;
    job.species = species;
    job.nnz = row_ptr[species];
    job.row_ptr = row_ptr;
    job.col_idx = col_idx;
    job.values = values;
    job.rhs = rhs;
    job.tol = tol;
    job.max_iter = max_iter;
    job.x_out = x_out;
    job.n_groups = n_groups;
    job.g_begin = gb;
    job.g_end = ge;
    job.block_width = block_width;
    job.g_iters = group_iters;
    job.g_rms = group_rms;
    job.g_flags = group_flags;
    job.status = ORC_OK;
    pthread_mutex_init(&job.lock, NULL);

    if (workers < 1) workers = 1;
    if (workers > n_groups) workers = n_groups;
    if (workers <= 1) {
        batch_worker(&job);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
        for (int64_t w = 0; w < workers; ++w) pthread_create(&th[w], NULL, batch_worker, &job);
        for (int64_t w = 0; w < workers; ++w) pthread_join(th[w], NULL);
        free(th);
    }
    pthread_mutex_destroy(&job.lock);
    st = job.status;
    if (st == ORC_OK && report) { /* strategies.cpp:71-87 merge_groups */
        memset(report, 0, sizeof *report);
        report->n_groups = n_groups;
        report->cells_per_block = cpb;
        for (int64_t g = 0; g < n_groups; ++g) {
            report->iterations_sum += group_iters[g];
            if (group_iters[g] > report->iterations_effective)
                report->iterations_effective = group_iters[g];
            if (group_rms[g] > report->max_residual_rms) report->max_residual_rms = group_rms[g];
            report->breakdown_fallbacks += (group_flags[g] & ORC_FLAG_FELL_BACK) ? 1 : 0;
        }
    }
    free(gb);
    free(ge);
    return st;
}
