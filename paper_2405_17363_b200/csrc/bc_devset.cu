// bc_devset.cu -- the drop-in API over several GPUs of one box.
//
// The reference parallelises solve_block_cells over a worker pool
// (strategies.cpp:221-247) and merges the groups in group order
// (merge_groups, strategies.cpp:71-87).  Here the workers are GPUs: a device
// set holds one bc_ctx per device, shards a batch into contiguous,
// group-aligned cell ranges (the leftover group, strategies.cpp:209-213,
// stays on the last shard), and runs one host thread per device, each
// calling bc_solve on its own context and stream.  Every group is the group
// a single-GPU run forms, so x, per-group iterations / rms / flags are
// bit-identical to bc_solve on one device; the shards write disjoint slices
// of the caller's arrays, and the SolveReport scalars are merged in shard
// (= group) order exactly as merge_groups folds them.  No collective: cells
// are independent.  Multi-cells is one global system with global scalars and
// runs on the set's first device only (replicas-only).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "blockcells_b200.h"

struct bc_devset {
    std::vector<bc_ctx*> ctx;
    std::vector<int> device;
    std::vector<cudaStream_t> stream;
    std::string err;
};

namespace {

bool host_pointer(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return true;
    }
    return a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged;
}

// Contiguous group-aligned shard of a batch (paper_2405_17363_b200/sharding.py
// shard_range): groups [g0, g1) of the full groups, plus the leftover group on
// the last shard.
void shard(int64_t cells, int64_t k, int rank, int world, int64_t* first, int64_t* count) {
    const int64_t full = cells / k, rem = cells % k;
    const int64_t per = full / world, extra = full % world;
    const int64_t g0 = rank * per + std::min<int64_t>(rank, extra);
    const int64_t g1 = g0 + per + (rank < extra ? 1 : 0);
    int64_t last = g1 * k;
    if (rank == world - 1) last += rem;
    *first = g0 * k;
    *count = last - g0 * k;
}

}  // namespace

extern "C" {

int bc_devset_create(int n_devices, const int* devices, bc_devset** out) {
    if (!out || n_devices < 1 || !devices) return BC_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    bc_devset* s = new (std::nothrow) bc_devset;
    if (!s) return BC_ERR_NO_MEMORY;
    for (int i = 0; i < n_devices; ++i) {
        bc_ctx* c = nullptr;
        int st = bc_ctx_create(devices[i], &c);
        cudaStream_t strm = nullptr;
        if (st == BC_OK && (cudaSetDevice(devices[i]) != cudaSuccess ||
                            cudaStreamCreateWithFlags(&strm, cudaStreamNonBlocking) != cudaSuccess))
            st = BC_ERR_CUDA;
        if (st != BC_OK) {
            if (c) bc_ctx_destroy(c);
            bc_devset_destroy(s);
            return st;
        }
        s->ctx.push_back(c);
        s->device.push_back(devices[i]);
        s->stream.push_back(strm);
    }
    *out = s;
    return BC_OK;
}

void bc_devset_destroy(bc_devset* s) {
    if (!s) return;
    for (size_t i = 0; i < s->ctx.size(); ++i) {
        if (s->stream[i]) {
            cudaSetDevice(s->device[i]);
            cudaStreamDestroy(s->stream[i]);
        }
        bc_ctx_destroy(s->ctx[i]);
    }
    delete s;
}

int bc_devset_size(const bc_devset* s) { return s ? static_cast<int>(s->ctx.size()) : 0; }

const char* bc_devset_last_error(const bc_devset* s) { return s ? s->err.c_str() : "null device set"; }

int bc_devset_set_pattern(bc_devset* s, int32_t species, const int32_t* row_ptr, const int32_t* col_idx) {
    if (!s) return BC_ERR_INVALID_ARGUMENT;
    s->err.clear();
    for (bc_ctx* c : s->ctx) {
        const int st = bc_set_pattern(c, species, row_ptr, col_idx);
        if (st != BC_OK) {
            s->err = bc_last_error(c);
            return st;
        }
    }
    return BC_OK;
}

int bc_devset_solve(bc_devset* s, const bc_solve_params* prm, const double* values, const double* rhs,
                    double* x_out, int32_t* group_iters, double* group_rms, uint8_t* group_flags,
                    bc_report* report) {
    if (!s || !prm) return BC_ERR_INVALID_ARGUMENT;
    s->err.clear();
    const int world = static_cast<int>(s->ctx.size());
    bc_ctx* c0 = s->ctx[0];
    // the pattern's size, from a plan query on the first context's pattern
    int64_t n_groups = 0;
    double cpb = 0.0;
    int32_t species = 0, nnz = 0;
    {
        // bc_plan needs the species; the contexts share one pattern
        int32_t info[2] = {0, 0};
        const int st = bc_ctx_pattern_info(c0, info);
        if (st != BC_OK) {
            s->err = bc_last_error(c0);
            return st;
        }
        species = info[0];
        nnz = info[1];
    }
    int st = bc_plan(species, prm, &n_groups, &cpb);
    if (st != BC_OK) {
        s->err = "bc_plan failed";
        return st;
    }
    const bool multi = prm->strategy == BC_STRATEGY_MULTI_CELLS;
    const int use = multi ? 1 : world;
    if (use > 1 && (!host_pointer(values) || !host_pointer(rhs) || !host_pointer(x_out))) {
        s->err = "a device-set solve over several GPUs takes host arrays (pageable or pinned)";
        return BC_ERR_INVALID_ARGUMENT;
    }
    const int64_t k = prm->strategy == BC_STRATEGY_BLOCK_CELLS ? static_cast<int64_t>(cpb) : 1;
    std::vector<int64_t> first(use, 0), count(use, prm->cells), g0(use, 0);
    if (!multi)
        for (int r = 0; r < use; ++r) {
            shard(prm->cells, k, r, use, &first[r], &count[r]);
            g0[r] = first[r] / k;
        }
    std::vector<bc_report> rep(use);
    std::vector<int> status(use, BC_OK);
    auto run = [&](int r) {
        if (count[r] == 0) return;
        bc_solve_params sub = *prm;
        sub.cells = count[r];
        if (use > 1 || !prm->stream) sub.stream = s->stream[r];  // one device: the caller's stream if given
        status[r] = bc_solve(s->ctx[r], &sub, values + first[r] * nnz, rhs + first[r] * species,
                             x_out + first[r] * species, group_iters ? group_iters + g0[r] : nullptr,
                             group_rms ? group_rms + g0[r] : nullptr, group_flags ? group_flags + g0[r] : nullptr,
                             &rep[r]);
    };
    if (use == 1) {
        run(0);
    } else {
        std::vector<std::thread> pool;
        for (int r = 0; r < use; ++r) pool.emplace_back(run, r);
        for (std::thread& t : pool) t.join();
    }
    for (int r = 0; r < use; ++r)
        if (status[r] != BC_OK) {
            s->err = "device " + std::to_string(s->device[r]) + ": " + bc_last_error(s->ctx[r]);
            return status[r];
        }
    if (report) {  // merge_groups (strategies.cpp:71-87), shards in group order
        std::memset(report, 0, sizeof *report);
        report->n_groups = n_groups;
        report->cells_per_block = cpb;
        for (int r = 0; r < use; ++r) {
            if (count[r] == 0) continue;
            const bc_report& q = rep[r];
            report->iterations_sum += q.iterations_sum;
            report->iterations_effective = std::max(report->iterations_effective, q.iterations_effective);
            report->max_residual_rms = std::max(report->max_residual_rms, q.max_residual_rms);
            report->breakdown_fallbacks += q.breakdown_fallbacks;
            report->device_ms = std::max(report->device_ms, q.device_ms);
            report->kernel_launches += q.kernel_launches;
            report->kernels |= q.kernels;
            report->model_spmv_wavefronts = std::max(report->model_spmv_wavefronts, q.model_spmv_wavefronts);
        }
    }
    return BC_OK;
}

int bc_host_alloc(uint64_t bytes, void** out) {
    if (!out) return BC_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (bytes == 0) return BC_OK;
    // portable: pinned for every device of a set; mapped: the kernels can
    // write x straight into it (bc_solve's zero-copy output path)
    if (cudaHostAlloc(out, bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
        (void)cudaGetLastError();
        *out = nullptr;
        return BC_ERR_NO_MEMORY;
    }
    return BC_OK;
}

void bc_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
