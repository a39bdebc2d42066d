// Microbenchmark: throughput of scattered per-lane 32-byte gathers from an
// L2-resident table through the different load paths (tuning aid for the
// ensemble walks: K4 on config #4 is bound by L1/TEX wavefronts of scattered
// block loads, one per distinct 128-byte line per warp instruction).
// Each thread runs CHAINS independent pointer-chasing chains (the next index
// comes from the loaded data, like a tree walk) for STEPS steps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef CHAINS
#define CHAINS 8
#endif
constexpr int STEPS = 256;

__device__ __forceinline__ void ld256(const void *p, uint32_t (&w)[8]) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                   "=r"(w[6]), "=r"(w[7]) : "l"(p));
}

template <int MODE>
__global__ void chase(const uint4 *tab, cudaTextureObject_t tex, uint32_t mask, uint32_t *out) {
    uint32_t idx[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) idx[c] = ((blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + c * 40503u) & mask;
    uint32_t acc = 0;
    for (int s = 0; s < STEPS; s++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            uint32_t a, b;
            if (MODE == 0) {          // one 256-bit LDG per block
                uint32_t w[8];
                ld256(tab + 2 * (size_t)idx[c], w);
                a = w[0] ^ w[5]; b = w[7];
            } else if (MODE == 1) {   // one 128-bit LDG (half block)
                const uint4 v = __ldg(tab + 2 * (size_t)idx[c]);
                a = v.x ^ v.y; b = v.w;
            } else if (MODE == 2) {   // texture path, one 128-bit fetch
                const uint4 v = tex1Dfetch<uint4>(tex, 2 * idx[c]);
                a = v.x ^ v.y; b = v.w;
            } else {                  // 64-bit LDG
                const uint2 v = __ldg(reinterpret_cast<const uint2 *>(tab + 2 * (size_t)idx[c]));
                a = v.x; b = v.y;
            }
            acc += b;
            idx[c] = (a * 2654435761u + idx[c]) & mask;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const size_t blocks = 1u << 20;  // 1M 32-byte blocks = 32 MB (L2-resident)
    uint4 *tab; uint32_t *out;
    cudaMalloc(&tab, blocks * 32); cudaMalloc(&out, 4);
    {
        uint32_t *h = (uint32_t *)malloc(blocks * 32);
        for (size_t i = 0; i < blocks * 8; i++) h[i] = (uint32_t)(i * 0x9E3779B9u) ^ (uint32_t)(i >> 7);
        cudaMemcpy(tab, h, blocks * 32, cudaMemcpyHostToDevice);
        free(h);
    }
    cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeLinear; rd.res.linear.devPtr = tab;
    rd.res.linear.desc = cudaCreateChannelDesc<uint4>(); rd.res.linear.sizeInBytes = blocks * 32;
    cudaTextureDesc td = {}; td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex; cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    int sm = 0; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char *names[4] = {"LDG.256", "LDG.128", "TEX.128", "LDG.64"};
    for (int threads : {128, 256}) for (int per_sm : {4, 8, 16}) for (int mode = 0; mode < 4; mode++) {
        const int grid = sm * per_sm;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        auto run = [&] {
            if (mode == 0) chase<0><<<grid, threads>>>(tab, tex, (uint32_t)blocks - 1, out);
            if (mode == 1) chase<1><<<grid, threads>>>(tab, tex, (uint32_t)blocks - 1, out);
            if (mode == 2) chase<2><<<grid, threads>>>(tab, tex, (uint32_t)blocks - 1, out);
            if (mode == 3) chase<3><<<grid, threads>>>(tab, tex, (uint32_t)blocks - 1, out);
        };
        run(); cudaDeviceSynchronize();
        cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        const double loads = (double)grid * threads * CHAINS * STEPS;
        const double cyc = ms * 1e-3 * clk * 1e3 * sm;  // SM-cycles at the nominal clock
        printf("%-8s threads %3d ctas/sm %2d chains %d: %7.3f ms  %6.2f G lane-loads/s  %5.2f lane-loads/SM-cycle\n",
               names[mode], threads, per_sm, CHAINS, ms, loads / ms / 1e6, loads / cyc);
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
