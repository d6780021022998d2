// Microbenchmark: MUFU (ex2 / rcp / tanh) and FFMA throughput per SM per clock on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float *out, int iters, long long *cyc) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (OP == 1) asm volatile("{.reg .f32 t; add.f32 t, %0, 0f3F800000; rcp.approx.ftz.f32 %0, t;}" : "+f"(a[i]));
            if (OP == 2) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a[i]));
            if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
            if (OP == 4) asm volatile("{.reg .f32 t; ex2.approx.ftz.f32 t, %0; add.f32 t, t, 0f3F800000; rcp.approx.ftz.f32 %0, t;}" : "+f"(a[i]));
            if (OP == 5) asm volatile("{.reg .f32 t; add.f32 t, %0, 0f3F800000; mul.f32 t, t, 0f3F000000; add.f32 %0, t, 0f3F800000;}" : "+f"(a[i]));
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float *out; long long *cyc;
    int blocks = 148, threads = 1024, iters = 4096;
    cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
    const char *names[6] = {"ex2", "rcp(+add)", "tanh", "ffma", "ex2+add+rcp", "add+mul+add"};
    for (int op = 0; op < 6; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, threads>>>(out, iters, cyc);
            if (op == 1) k<1><<<blocks, threads>>>(out, iters, cyc);
            if (op == 2) k<2><<<blocks, threads>>>(out, iters, cyc);
            if (op == 3) k<3><<<blocks, threads>>>(out, iters, cyc);
            if (op == 4) k<4><<<blocks, threads>>>(out, iters, cyc);
            if (op == 5) k<5><<<blocks, threads>>>(out, iters, cyc);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            double ops = (double)threads * iters * 8;   // per SM (one block per SM)
            if (rep) printf("%s: %.2f ops/clk/SM (cycles %lld), %.1f Gops/s total, %.3f ms\n", names[op], ops / h[0], h[0],
                            ops * blocks / ms / 1e6, ms);
        }
    }
    return 0;
}
