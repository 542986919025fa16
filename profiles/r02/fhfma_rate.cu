// FFMA vs mixed-precision fma.rn.f32.f16 (SASS FHFMA) issue rate on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fh fhfma_rate.cu && ./fh
// throughput of FFMA vs mixed f16xf16+f32 FMA (FHFMA) on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, unsigned a0, unsigned b0, int iters) {
    float acc[8];
    unsigned a[8];
    for (int j = 0; j < 8; ++j) { acc[j] = threadIdx.x * 1e-9f + j; a[j] = a0 + j * 77 + threadIdx.x; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (MODE == 0) {
                acc[j] = fmaf(__uint_as_float(a[j]), __uint_as_float(b0), acc[j]);
                acc[j] = fmaf(__uint_as_float(b0), __uint_as_float(a[j]), acc[j]);
            } else {
                asm volatile("{\n .reg .f16 x0, x1, y0, y1;\n mov.b32 {x0, x1}, %1;\n mov.b32 {y0, y1}, %2;\n"
                    " fma.rn.f32.f16 %0, x0, y0, %0;\n fma.rn.f32.f16 %0, x1, y1, %0;\n}"
                    : "+f"(acc[j]) : "r"(a[j]), "r"(b0));
            }
        }
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 512 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode) for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<148 * 4, 512>>>(out, 0x3c003c00u, 0x3c013c01u, iters);
        else k<1><<<148 * 4, 512>>>(out, 0x3c003c00u, 0x3c013c01u, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = 148.0 * 4 * 512 * iters * 16;
        printf("mode %d (%s): %.3f ms, %.1f G fma-instr/s per SM-clk-est %.2f /clk/SM\n", mode, mode ? "FHFMA" : "FFMA", ms,
               fmas / ms / 1e6, fmas / (ms * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
