// Micro-benchmark: do scalar FFMA and packed FFMA2 issue to separate pipes on sm_100a?
// Each thread runs 8 independent chains; variants: only FFMA2, only FFMA, FFMA2 + FFMA mixed.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float fma1(float a, float b, float c) {
    float r;
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
template <int NP, int NS>
__global__ void k(float* out, int iters, float s) {
    f2 p[8];
    float q[8];
    for (int i = 0; i < 8; ++i) {
        p[i] = (f2)(threadIdx.x + i);
        q[i] = threadIdx.x * 0.1f + i;
    }
    const f2 m = 0x3f8000003f800000ull;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int r = 0; r < NP; ++r) p[i] = fma2(p[i], m, m);
#pragma unroll
            for (int r = 0; r < NS; ++r) q[i] = fma1(q[i], s, s);
        }
    }
    float acc = 0;
    for (int i = 0; i < 8; ++i) acc += __uint_as_float((unsigned)p[i]) + q[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int NP, int NS>
void run(const char* name, float* d) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    k<NP, NS><<<148 * 4, 256>>>(d, iters, 1.0001f);
    cudaEventRecord(a);
    k<NP, NS><<<148 * 4, 256>>>(d, iters, 1.0001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr = 148.0 * 4 * 8 * iters * 8 * (NP + NS);  // warps x ...
    const double lane_flops = 148.0 * 4 * 256 * iters * 8 * (2.0 * NP * 2 + 2.0 * NS);
    printf("%-28s %8.3f ms  %7.1f TFLOP/s  %6.2f warp-instr/clk/SM (at 1.9 GHz)\n", name, ms,
           lane_flops / ms / 1e9, warp_instr / (ms * 1e-3) / 1.9e9 / 148);
}
int main() {
    float* d;
    cudaMalloc(&d, 148 * 4 * 256 * 4);
    run<4, 0>("FFMA2 x4", d);
    run<0, 8>("FFMA x8", d);
    run<0, 4>("FFMA x4", d);
    run<4, 4>("FFMA2 x4 + FFMA x4", d);
    run<4, 2>("FFMA2 x4 + FFMA x2", d);
    run<2, 4>("FFMA2 x2 + FFMA x4", d);
    return 0;
}
