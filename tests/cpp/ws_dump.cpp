// bicg_solve(..., BicgWorkspace& ws) on a few systems, printing every output
// bit the caller can see: x, iterations, flags, final rms and
// ws.per_block_error.  TEST INFRASTRUCTURE: built twice (tests/cpp/Makefile),
// over the B200 drop-in (ws_dump_b200) and over the reference's own bicg.o
// (ws_dump_reference); tests/test_dropin_overlap.py compares the two outputs.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "blockcells/bicg.hpp"
#include "blockcells/reduction.hpp"
#include "blockcells_workload.h"

using namespace blockcells;

static void put(const double* p, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) {
        uint64_t u;
        std::memcpy(&u, p + i, 8);
        std::printf("%016llx ", static_cast<unsigned long long>(u));
    }
}

int main() {
    const int cases[][4] = {  // species, block size of the reduction plan (0: one block), cells, max_iter
        {24, 0, 3, 400}, {40, 16, 2, 400}, {156, 64, 2, 1000}, {156, 100, 1, 7}, {60, 7, 2, 50}};
    for (const auto& c : cases) {
        const int species = c[0];
        bcw_mechanism* m = nullptr;
        if (bcw_mechanism_create(species, 3 * species, 1, &m) != 0) return 2;
        const long nnz = bcw_nnz(m);
        std::vector<int32_t> rp(species + 1), ci(nnz);
        bcw_pattern(m, rp.data(), ci.data());
        std::vector<double> vals(static_cast<size_t>(c[2]) * nnz), rhs(static_cast<size_t>(c[2]) * species);
        if (bcw_newton_batch(m, 0, c[2], c[2], 1, 60.0, nullptr, nullptr, vals.data(), rhs.data(), 0) != 0) return 3;
        ReductionPlan plan;
        if (c[1] == 0) {
            plan = ReductionPlan::single_block(species);
        } else {
            for (int b0 = 0; b0 < species; b0 += c[1])
                plan.block_ranges.push_back(IndexRange{static_cast<std::size_t>(b0),
                                                       static_cast<std::size_t>(std::min(species, b0 + c[1]))});
        }
        for (int cell = 0; cell < c[2]; ++cell) {
            CsrMatrix a;
            a.n_rows = a.n_cols = species;
            a.row_ptr.assign(rp.begin(), rp.end());
            a.col_idx.assign(ci.begin(), ci.end());
            a.values.assign(vals.begin() + cell * nnz, vals.begin() + (cell + 1) * nnz);
            DenseVector b(rhs.begin() + cell * species, rhs.begin() + (cell + 1) * species);
            DenseVector x0(species, 0.0);
            BicgWorkspace ws;
            const SolveOutcome o = bicg_solve(a, b, x0, 1e-12, static_cast<std::size_t>(c[3]), plan, ws);
            std::printf("case s=%d blk=%d cell=%d it=%zu conv=%d brk=%d rms=", species, c[1], cell, o.iterations,
                        o.converged ? 1 : 0, o.breakdown ? 1 : 0);
            put(&o.final_residual_rms, 1);
            std::printf("\nx ");
            put(o.x.data(), o.x.size());
            std::printf("\nper_block_error ");
            put(ws.per_block_error.data(), ws.per_block_error.size());
            std::printf("\n");
        }
        bcw_mechanism_destroy(m);
    }
    return 0;
}
