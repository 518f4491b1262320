// Phase profile of the shared-memory LU (bc_lu_sm.cuh built with
// BC_LU_PROFILE): cycles per 156 x 156 block of CTA 0's thread 0, on one
// Block-cells(k) group of the bench workload's Newton systems (P regime).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -DBC_LU_PROFILE
//     -I paper_2405_17363_b200/csrc -I include -o tools/luprof.bin tools/luprof.cu
//     -L paper_2405_17363_b200 -lbc_workload -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2405_17363_b200'
// usage: tools/luprof.bin [species=156] [k=6] [ctas=1]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bc_lu_sm.cuh"
#include "blockcells_workload.h"

int main(int argc, char** argv) {
    const int species = argc > 1 ? atoi(argv[1]) : 156;
    const int k = argc > 2 ? atoi(argv[2]) : 6;
    const int ctas = argc > 3 ? atoi(argv[3]) : 1;
    bcw_mechanism* m = nullptr;
    bcw_mechanism_create(species, 3 * species, 0, &m);
    const int nnz = static_cast<int>(bcw_nnz(m));
    std::vector<int32_t> rp(species + 1), ci(nnz);
    bcw_pattern(m, rp.data(), ci.data());
    const int cells = k * ctas;
    std::vector<double> vals(static_cast<size_t>(nnz) * cells), rhs(static_cast<size_t>(species) * cells);
    bcw_newton_batch(m, 0, cells, 100000, 1, 120.0, nullptr, nullptr, vals.data(), rhs.data(), 1);
    auto up = [](const void* h, size_t b) { void* d; cudaMalloc(&d, b); cudaMemcpy(d, h, b, cudaMemcpyHostToDevice); return d; };
    std::vector<bc::LuEntry> ents(ctas);
    for (int i = 0; i < ctas; ++i) ents[i] = {static_cast<int64_t>(i) * k, i, k, 0};
    bc::LuParams p{};
    p.values = (const double*)up(vals.data(), 8 * vals.size());
    p.rhs = (const double*)up(rhs.data(), 8 * rhs.size());
    cudaMalloc(&p.x_out, 8 * rhs.size());
    cudaMalloc(&p.g_rms, 8 * ctas);
    cudaMalloc(&p.status, 4 * ctas);
    p.entries = (const bc::LuEntry*)up(ents.data(), sizeof(bc::LuEntry) * ctas);
    p.row_ptr = (const int32_t*)up(rp.data(), 4 * rp.size());
    p.col_idx = (const int32_t*)up(ci.data(), 4 * ci.size());
    p.stride = static_cast<int64_t>(k) * species * species;
    cudaMalloc(&p.scratch, 8 * p.stride * ctas);
    p.species = species;
    p.nnz = nnz;
    const size_t smem = bc::lu_sm_factor_smem(species);
    cudaFuncSetAttribute(bc::lu_sm_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const char* names[14] = {"panel", "row swaps", "U12", "A22", "densify", "factor total", "checks",
                             "forward", "park factors", " panel: bar", " panel: scan+pivot", " panel: update+publish",
                             " panel: scan (loads+local)", " -"};
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[64] = {0};
        cudaMemcpyToSymbol(bc::bc_lu_prof, z, sizeof z);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        bc::lu_sm_factor_kernel<<<ctas, bc::kLuSmThreads, smem>>>(p);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[64];
        cudaMemcpyFromSymbol(h, bc::bc_lu_prof, sizeof h);
        int st = 0;
        cudaMemcpy(&st, p.status, 4, cudaMemcpyDeviceToHost);
        printf("rep %d: %d CTAs x %d blocks, %.3f ms, status %d (%s)\n", rep, ctas, k, ms, st,
               cudaGetErrorString(cudaGetLastError()));
        for (int i = 0; i < 9; ++i) printf("  %-16s %10.0f cycles/block\n", names[i], double(h[i]) / k);
        for (int w = 0; w < 12; ++w)
            if (h[16 + 4 * w] + h[17 + 4 * w] + h[18 + 4 * w] + h[19 + 4 * w])
                printf("  warp %2d panel: bar-return %8.0f  pivot %8.0f  update %8.0f  scan %8.0f\n", w,
                       double(h[16 + 4 * w]) / k, double(h[17 + 4 * w]) / k, double(h[18 + 4 * w]) / k,
                       double(h[19 + 4 * w]) / k);
    }
    return 0;
}
