// Microbenchmark: throughput of fp32->fp16x2 packing (F2FP), LOP3, FADD, and cvt variants per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(uint32_t *out, int iters, long long *cyc) {
    float a[8]; uint32_t u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i * 1e-4f; u[i] = threadIdx.x + i; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "+r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
            if (OP == 1) asm volatile("and.b32 %0, %0, 0xFFFFE000;" : "+r"(u[i]));
            if (OP == 2) asm volatile("add.f32 %0, %0, %0;" : "+f"(a[i]));
            if (OP == 3) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
            if (OP == 4) asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(*(unsigned short *)&u[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
            if (OP == 5) asm volatile("{.reg .f16x2 h; mov.b32 h, %0; fma.rn.f16x2 h, h, h, h; mov.b32 %0, h;}" : "+r"(u[i]));
        }
        if (OP == 0 || OP == 3 || OP == 4) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __uint_as_float(u[i]);
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += u[i] + __float_as_uint(a[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    uint32_t *out; long long *cyc;
    int blocks = 148, threads = 1024, iters = 2048;
    cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
    const char *names[6] = {"cvt.rn.f16x2.f32 (F2FP)", "and.b32 (LOP3)", "add.f32", "cvt.rn.bf16x2.f32", "cvt e4m3x2", "fma.f16x2"};
    for (int op = 0; op < 6; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            if (op == 0) k<0><<<blocks, threads>>>(out, iters, cyc);
            if (op == 1) k<1><<<blocks, threads>>>(out, iters, cyc);
            if (op == 2) k<2><<<blocks, threads>>>(out, iters, cyc);
            if (op == 3) k<3><<<blocks, threads>>>(out, iters, cyc);
            if (op == 4) k<4><<<blocks, threads>>>(out, iters, cyc);
            if (op == 5) k<5><<<blocks, threads>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            double ops = (double)threads * iters * 8;
            if (rep) printf("%-26s %.2f ops/clk/SM\n", names[op], ops / h[0]);
        }
    }
    return 0;
}
