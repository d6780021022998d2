// Microbenchmark + layout check: tcgen05.mma kind::f16 with the A operand in TMEM ("TS") vs in shared
// memory ("SS"), M = 128.
//  check:  A (128 x 64 fp16) stored into TMEM with tcgen05.st, lane = row, 32-bit column j holding
//          K elements (2j, 2j+1); B (N x 64) in shared memory (SWIZZLE_128B, K-major); D = A B^T by
//          four K = 16 MMAs; compared with a host reference.
//  rate:   one CTA per SM, one thread issues R back-to-back MMAs (N = 256, K = 16), SS or TS, optionally
//          with 8 other warps streaming shared memory (ld.shared.v4) to load the SMEM crossbar.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_ts mma_ts.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(id),
                 "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(b), "r"(id),
                 "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n}" ::"r"(
                     smem_u32(bar)), "r"(ph) : "memory");
}

// ---- layout check: 1 CTA, 128 threads
__global__ void k_check(const __half *A, const __half *B, float *D, int N) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    // B: N rows x 64 K, SWIZZLE_128B K-major: byte r*128 + ((k/8 ^ r%8)*16) + (k%8)*2
    for (int e = t; e < N * 64; e += blockDim.x) {
        const int r = e / 64, k = e % 64;
        *(__half *)(sm + r * 128 + ((((k >> 3) ^ (r & 7)) << 4)) + (k & 7) * 2) = B[e];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    // A row t -> TMEM lane t, columns 256 + j: {A[t][2j], A[t][2j+1]}
    {
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) {
            __half2 h = __halves2half2(A[t * 64 + 2 * j], A[t * 64 + 2 * j + 1]);
            r[j] = *(uint32_t *)&h;
        }
        const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + 256;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                     "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                     "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                     "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
        const uint32_t id = idesc_f16(128, N);
        for (int kk = 0; kk < 4; ++kk)   // K = 16 per MMA = 8 TMEM columns of A, 32 bytes of each B row
            mma_ts(tm, tm + 256 + 8 * kk, sdesc_sw128(smem_u32(sm) + kk * 32, 16, 1024), id, kk > 0);
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < N; c += 16) {
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) D[t * N + c + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// ---- rate: per CTA R MMAs M128 N256 K16; mode 0 SS, 1 TS; noise: extra warps streaming shared memory
__global__ void k_rate(int R, int mode, int noise, long long *cyc, float *sink) {
    extern __shared__ __align__(1024) uint8_t sm[];   // 64 KB: A (16 KB) + B (32 KB) + noise area
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ volatile int done;
    const int t = threadIdx.x, warp = t >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); done = 0; }
    for (int e = t; e < 65536 / 4; e += blockDim.x) ((uint32_t *)sm)[e] = 0x3C003C00u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    if (t == 0) {
        const uint32_t id = idesc_f16(128, 256);
        const uint32_t a = smem_u32(sm), b = smem_u32(sm) + 16384;
        long long t0 = clock64();
        for (int i = 0; i < R; ++i) {
            const int kk = i & 3;
            if (mode == 0) mma_ss(tm, sdesc_sw128(a + kk * 32, 16, 1024), sdesc_sw128(b + kk * 32, 16, 1024), id, 1);
            else mma_ts(tm, tm + 256 + 8 * kk, sdesc_sw128(b + kk * 32, 16, 1024), id, 1);
        }
        commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
        done = 1;
    } else if (noise && warp >= 1) {
        uint32_t acc = 0;
        const uint32_t base = smem_u32(sm) + 49152 + (t & 255) * 16;
        while (!done) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                uint32_t x0, x1, x2, x3;
                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(base));
                acc += x0 ^ x1 ^ x2 ^ x3;
            }
        }
        if (acc == 12345) sink[t] = 1.0f;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    // layout check
    for (int N : {64, 128, 256}) {
        std::vector<__half> A(128 * 64), B(N * 64);
        std::vector<float> Af(128 * 64), Bf(N * 64);
        srand(1 + N);
        for (int i = 0; i < 128 * 64; ++i) { Af[i] = (float)((rand() % 17) - 8) / 8.0f; A[i] = __float2half(Af[i]); }
        for (int i = 0; i < N * 64; ++i) { Bf[i] = (float)((rand() % 13) - 6) / 4.0f; B[i] = __float2half(Bf[i]); }
        __half *dA, *dB;
        float *dD;
        cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, 128 * N * 4);
        cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        k_check<<<1, 128, 64 * 1024>>>(dA, dB, dD, N);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(128 * N);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0;
                for (int k = 0; k < 64; ++k) s += (double)Af[m * 64 + k] * Bf[n * 64 + k];
                maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
            }
        printf("TS layout check N=%d: %s max|err| = %g\n", N, cudaGetErrorString(e), maxerr);
    }
    // rates
    long long *dc;
    float *sink;
    int nsm = 148;
    cudaMalloc(&dc, nsm * 8); cudaMalloc(&sink, 1024 * 4);
    cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int noise = 0; noise <= 1; ++noise)
        for (int mode = 0; mode <= 1; ++mode) {
            const int R = 4096;
            k_rate<<<nsm, noise ? 288 : 32, 64 * 1024>>>(R, mode, noise, dc, sink);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<long long> c(nsm);
            cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto x : c) avg += x;
            avg /= nsm;
            printf("%s %s: %.1f cycles per M128 N256 K16 MMA (floor 128)  [%s]\n", mode ? "TS" : "SS",
                   noise ? "with 8 warps streaming ld.shared.v4" : "alone", avg / R, cudaGetErrorString(e));
        }
    return 0;
}
