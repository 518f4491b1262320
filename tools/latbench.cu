// Dependent-chain latencies on one B200 SM (single warp unless noted), in
// cycles per operation: DADD, DMUL, DDIV (__ddiv_rn), fp64 SHFL (two 32-bit
// shuffles + the add of a butterfly level), LDS.64 pointer chase, and an
// 8-warp bar.sync round.  Bounds the latency kernel (bc_latency.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o latbench tools/latbench.cu
#include <cstdio>
#include <cstdint>

__global__ void chains(double* out, long long* cyc, int n, double a, double b) {
    __shared__ double sm[1024];
    __shared__ uint32_t nxt[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i; nxt[i] = (i * 97 + 13) & 1023; }
    __syncthreads();
    double x = a + threadIdx.x * 1e-3, y = b;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __dadd_rn(x, y); x = __dadd_rn(x, y); x = __dadd_rn(x, y); x = __dadd_rn(x, y); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __dmul_rn(x, y); x = __dmul_rn(x, y); x = __dmul_rn(x, y); x = __dmul_rn(x, y); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
    // DDIV chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __ddiv_rn(x, y); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) * 4;
    // butterfly level: x += shfl_xor(x)
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 16)); x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 8));
        x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 4)); x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 2));
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
    // LDS.64 chase
    uint32_t k = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { k = nxt[k]; k = nxt[k]; k = nxt[k]; k = nxt[k]; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
    // bar.sync rounds (all warps of the block)
    t0 = clock64();
    for (int i = 0; i < n; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
    // STS + bar + LDS round (the reduction's shared step)
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        sm[threadIdx.x] = x; __syncthreads(); x = __dadd_rn(x, sm[(threadIdx.x + 32) & 1023]); __syncthreads();
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) * 4;
    out[threadIdx.x] = x + sm[k & 1023];
}

int main() {
    double* out; long long* cyc; long long h[8];
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 64);
    const char* names[7] = {"dadd", "dmul", "ddiv", "shfl64+dadd", "lds chase (u32)", "bar.sync", "sts+bar+lds+dadd+bar"};
    for (int threads : {32, 256}) {
        const int n = 2000;
        chains<<<1, threads>>>(out, cyc, n, 1.0000001, 0.9999999);
        chains<<<1, threads>>>(out, cyc, n, 1.0000001, 0.9999999);
        cudaMemcpy(h, cyc, 56, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 7; ++i) printf("threads=%d %-22s %.1f cycles/op\n", threads, names[i], h[i] / (4.0 * n));
    }
    return 0;
}
