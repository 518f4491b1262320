// End-to-end through the reference's own C++ entry point on the B200 drop-in:
// blockcells::run_strategy (strategies.hpp:80-82; the shim,
// paper_2405_17363_b200/shim/blockcells_b200_shim.cpp) on a BatchedSystem
// built the reference's way -- one CsrMatrix (own row_ptr/col_idx/values)
// and one DenseVector rhs per cell, strategies.hpp:15-23 -- so the timed call
// includes BatchedSystem::check, packing into the C ABI's flat arrays, the
// host->device streaming, the solve and the per-cell DenseVector outputs,
// exactly what the reference's caller (run_simulation, simulate.cpp:137-140)
// pays.  Inputs: the bench workload (M156, first Newton system of step 0,
// realistic conditions over the global cell index, P regime) from
// libbc_workload.  Prints one JSON line.  Algorithm: BLOCKCELLS_B200_ALGO
// (bicgstab | unset = BiCG); devices: BLOCKCELLS_B200_DEVICES (shim).
//   dropin_bench <cells> <steps> <warmup> [species] [h] [tol] [max_iter] [workers]
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include "blockcells/strategies.hpp"
#include "blockcells_workload.h"

using namespace blockcells;

int main(int argc, char** argv) {
    const long cells = argc > 1 ? atol(argv[1]) : 100000;
    const int steps = argc > 2 ? atoi(argv[2]) : 5;
    const int warmup = argc > 3 ? atoi(argv[3]) : 2;
    const int species = argc > 4 ? atoi(argv[4]) : 156;
    const double h = argc > 5 ? atof(argv[5]) : 120.0;        // P regime by default (bench.hpp:20)
    const double tol = argc > 6 ? atof(argv[6]) : 1e-30;
    const std::size_t max_iter = argc > 7 ? static_cast<std::size_t>(atol(argv[7])) : 1000;
    const std::size_t workers = argc > 8 ? static_cast<std::size_t>(atol(argv[8])) : 0;
    bcw_mechanism* m = nullptr;
    if (bcw_mechanism_create(species, 3 * species, 0, &m) != 0) return 2;
    const long nnz = bcw_nnz(m);
    std::vector<int32_t> rp(species + 1), ci(nnz);
    bcw_pattern(m, rp.data(), ci.data());
    std::vector<double> vals(static_cast<size_t>(cells) * nnz), rhs(static_cast<size_t>(cells) * species);
    if (bcw_newton_batch(m, 0, cells, cells, 1, h, nullptr, nullptr, vals.data(), rhs.data(), 0) != 0) return 3;
    BatchedSystem sys;
    sys.species = species;
    sys.cells = cells;
    CsrMatrix proto;
    proto.n_rows = proto.n_cols = species;
    proto.row_ptr.assign(rp.begin(), rp.end());
    proto.col_idx.assign(ci.begin(), ci.end());
    sys.per_cell_matrices.reserve(cells);
    sys.per_cell_rhs.reserve(cells);
    for (long c = 0; c < cells; ++c) {
        CsrMatrix a = proto;
        a.values.assign(vals.begin() + c * nnz, vals.begin() + (c + 1) * nnz);
        sys.per_cell_matrices.push_back(std::move(a));
        sys.per_cell_rhs.emplace_back(rhs.begin() + c * species, rhs.begin() + (c + 1) * species);
    }
    vals.clear();
    vals.shrink_to_fit();
    // error-path checks (tests/test_dropin_overlap.py): a cell whose pattern
    // differs and/or a cell whose rhs has the wrong size; run_strategy must
    // throw what BatchedSystem::check (strategies.cpp:91-107) throws
    const char* bad_pat = std::getenv("DROPIN_BAD_PATTERN_CELL");
    const char* bad_rhs = std::getenv("DROPIN_BAD_RHS_CELL");
    if (bad_pat || bad_rhs) {
        if (bad_pat) std::swap(sys.per_cell_matrices[atol(bad_pat)].col_idx[0], sys.per_cell_matrices[atol(bad_pat)].col_idx[1]);
        if (bad_rhs) sys.per_cell_rhs[atol(bad_rhs)].resize(species - 1);
        StrategyConfig c1;
        c1.kind = Strategy::BlockCells;
        c1.cells_per_block = 1;
        try {
            run_strategy(sys, c1, DeviceSpec{}, tol, max_iter, workers);
            std::printf("{\"error\": null}\n");
        } catch (const std::invalid_argument& e) {
            std::printf("{\"error\": \"%s\"}\n", e.what());
        }
        bcw_mechanism_destroy(m);
        return 0;
    }
    StrategyConfig cfg;
    cfg.kind = Strategy::BlockCells;
    cfg.cells_per_block = 1;
    double total = 0.0, rep_total = 0.0;
    std::size_t it_sum = 0, fallbacks = 0;
    uint64_t digest = 0;
    for (int i = 0; i < warmup + steps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        const SolveReport r = run_strategy(sys, cfg, DeviceSpec{}, tol, max_iter, workers);
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (i >= warmup) {
            total += dt;
            rep_total += r.wall_time_ns * 1e-9;
            it_sum = r.iterations_sum;
            fallbacks = r.breakdown_fallbacks;
            // FNV-1a over every output bit: x of every cell, per-group
            // iterations, the report's max rms and effective iterations
            uint64_t h = 1469598103934665603ull;
            auto mix = [&](const void* p, std::size_t n) {
                const unsigned char* b = static_cast<const unsigned char*>(p);
                for (std::size_t q = 0; q < n; ++q) h = (h ^ b[q]) * 1099511628211ull;
            };
            for (const auto& xc : r.per_cell_x) mix(xc.data(), sizeof(double) * xc.size());
            for (std::size_t g : r.per_block_iterations) mix(&g, sizeof g);
            mix(&r.max_residual_rms, sizeof r.max_residual_rms);
            mix(&r.iterations_effective, sizeof r.iterations_effective);
            mix(&r.iterations_sum, sizeof r.iterations_sum);
            digest = h;
        }
    }
    const char* algo = std::getenv("BLOCKCELLS_B200_ALGO");
    std::printf("{\"cells\": %ld, \"species\": %d, \"steps\": %d, \"warmup\": %d, \"algorithm\": \"%s\", "
                "\"h\": %g, \"tol\": %g, \"max_iter\": %zu, \"value\": %.3f, \"unit\": \"cell-solves/s\", \"ms_per_step\": %.3f, "
                "\"report_wall_ms_per_step\": %.3f, \"iterations_sum\": %zu, \"breakdown_fallbacks\": %zu, "
                "\"entry\": \"blockcells::run_strategy (strategies.hpp:80-82) over the drop-in shim\", "
                "\"input_bytes_per_step\": %ld, \"output_digest\": \"%016llx\"}\n",
                cells, species, steps, warmup, algo ? algo : "bicg", h, tol, max_iter, cells * steps / total, 1e3 * total / steps,
                1e3 * rep_total / steps, it_sum, fallbacks, static_cast<long>(cells) * (nnz + species) * 8,
                static_cast<unsigned long long>(digest));
    bcw_mechanism_destroy(m);
    return 0;
}
