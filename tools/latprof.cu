// Phase profile of the latency kernel on the bench workload's M156 cell:
// cycles per Jacobi-BiCGSTAB iteration phase (bc_latency.cuh built with
// BC_LAT_PROFILE), CTA 0 thread 0, P regime (1000 iterations).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 --extended-lambda
//     -DBC_LAT_PROFILE -I paper_2405_17363_b200/csrc -I include -o tools/latprof.bin tools/latprof.cu
//     paper_2405_17363_b200/csrc/bc_latency_plan.cpp paper_2405_17363_b200/csrc/bc_plan.cpp
//     -L paper_2405_17363_b200 -lbc_workload -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2405_17363_b200'
#include <cstdio>
#include <vector>

#include "bc_latency.cuh"
#include "bc_plan.hpp"
#include "blockcells_workload.h"

double sigma_max_for(double tol, int n);  // below

int main(int argc, char** argv) {
    const int species = argc > 1 ? atoi(argv[1]) : 156;
    bcw_mechanism* m = nullptr;
    bcw_mechanism_create(species, 3 * species, 0, &m);
    const int nnz = static_cast<int>(bcw_nnz(m));
    bc::Pattern pat;
    pat.species = species;
    pat.nnz = nnz;
    pat.row_ptr.resize(species + 1);
    pat.col_idx.resize(nnz);
    bcw_pattern(m, pat.row_ptr.data(), pat.col_idx.data());
    pat.diag.assign(species, -1);
    for (int i = 0; i < species; ++i)
        for (int e = pat.row_ptr[i]; e < pat.row_ptr[i + 1]; ++e)
            if (pat.col_idx[e] == i) pat.diag[i] = e;
    std::vector<double> vals(nnz), rhs(species);
    bcw_newton_batch(m, 0, 1, 100000, 1, 120.0, nullptr, nullptr, vals.data(), rhs.data(), 1);
    const bc::LatencySchedule ls = bc::build_latency_schedule(pat, 1, false, 160);
    auto up = [](const void* h, size_t b) { void* d; cudaMalloc(&d, b); cudaMemcpy(d, h, b, cudaMemcpyHostToDevice); return d; };
    bc::LatencyParams p{};
    p.values = (double*)up(vals.data(), 8 * nnz);
    p.rhs = (double*)up(rhs.data(), 8 * species);
    cudaMalloc(&p.x_out, 8 * species);
    cudaMalloc(&p.g_iters, 4); cudaMalloc(&p.g_rms, 8); cudaMalloc(&p.g_flags, 1);
    p.rowof = (int32_t*)up(ls.rowof.data(), 4 * ls.T);
    p.steps = (int32_t*)up(ls.steps.data(), 4 * ls.T);
    p.rvi = (int32_t*)up(ls.rvi.data(), 4 * ls.rvi.size());
    p.rxo = (uint16_t*)up(ls.rxo.data(), 2 * ls.rxo.size());
    p.didx = (int32_t*)up(ls.didx.data(), 4 * ls.P);
    p.group_count = 1; p.n = species; p.nnz = nnz; p.P = ls.P; p.species = species; p.kc = 1; p.xs = ls.xslots;
    p.sigma_max = 0.0; p.tol = 1e-30; p.max_iter = 1000;
    const size_t smem = 8 * (4 * ls.P + 5 * ls.xslots);
    printf("P=%d T=%d L=%d model gathers/SpMV=%d\n", ls.P, ls.T, ls.L, ls.model_wavefronts);
    if (ls.P != 256 || ls.L != 24) { printf("instance not compiled here\n"); return 1; }
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(bc::bc_lat_prof, z, sizeof z);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        bc::block_cells_latency_kernel<8, 5, 24, 1><<<1, ls.T, smem>>>(p);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[16];
        cudaMemcpyFromSymbol(h, bc::bc_lat_prof, sizeof h);
        int it; cudaMemcpy(&it, p.g_iters, 4, cudaMemcpyDeviceToHost);
        if (rep == 0) continue;
        const char* nm[9] = {"beta,p,y", "spmv(y)", "reduce den", "alpha,s,z,x", "spmv(z)", "reduce tt,ts", "omega,x,r", "reduce sigma,rho", "checks"};
        double tot = 0;
        for (int i = 0; i < 9; ++i) tot += h[i];
        for (int i = 0; i < 9; ++i) printf("%-26s %8.1f cycles/iter\n", nm[i], double(h[i]) / it);
        printf("total %.1f cycles/iter over %d iterations; kernel %.3f ms (%s)\n", tot / it, it, ms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
