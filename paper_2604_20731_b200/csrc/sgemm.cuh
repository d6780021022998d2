// sgemm.cuh -- fp32 SIMT (FFMA) tiled GEMM with pluggable epilogues.
// Used by the CRVPINN_PREC_FP32 MLP path and by the fp32 sine-transform Gram solve.
// C[M x N] = A[M x K] B[K x N]; A(m,k) = TA ? A[k*lda+m] : A[m*lda+k];
// B(k,n) = TB ? B[n*ldb+k] : B[k*ldb+n]. blockIdx.z selects a K-chunk (split-K).
#pragma once
#include "common.cuh"

namespace crv {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

template <bool TA, bool TB, class Epi>
__global__ void __launch_bounds__(256)
k_sgemm(int M, int N, int K, const float *__restrict__ A, int lda, const float *__restrict__ B,
        int ldb, int kchunk, Epi epi) {
    __shared__ float As[SG_BK][SG_BM + 4];
    __shared__ float Bs[SG_BK][SG_BN + 4];
    const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
    const int kbeg = blockIdx.z * kchunk;
    const int kend = min(K, kbeg + kchunk);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

    for (int k0 = kbeg; k0 < kend; k0 += SG_BK) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int e = tid + r * 256;
            int mm, kk;
            if (TA) { kk = e >> 6; mm = e & 63; } else { mm = e >> 4; kk = e & 15; }
            int gm = m0 + mm, gk = k0 + kk;
            float v = 0.0f;
            if (gm < M && gk < kend) v = TA ? A[(long)gk * lda + gm] : A[(long)gm * lda + gk];
            As[kk][mm] = v;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int e = tid + r * 256;
            int nn, kk;
            if (TB) { nn = e >> 4; kk = e & 15; } else { kk = e >> 6; nn = e & 63; }
            int gn = n0 + nn, gk = k0 + kk;
            float v = 0.0f;
            if (gn < N && gk < kend) v = TB ? B[(long)gn * ldb + gk] : B[(long)gk * ldb + gn];
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < SG_BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
            if (m < M && n < N) epi(m, n, acc[i][j], (int)blockIdx.z);
        }
}

template <bool TA, bool TB, class Epi>
void sgemm(int M, int N, int K, const float *A, int lda, const float *B, int ldb, int nsplit,
           Epi epi, cudaStream_t s) {
    int kchunk = K;
    if (nsplit > 1) {
        kchunk = ceil_div(ceil_div(K, nsplit), SG_BK) * SG_BK;
        nsplit = ceil_div(K, kchunk);
    }
    dim3 grid(ceil_div(N, SG_BN), ceil_div(M, SG_BM), nsplit);
    k_sgemm<TA, TB, Epi><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, kchunk, epi);
}

// Split count actually used by sgemm() for a requested nsplit (for partial-buffer planning).
inline int sgemm_effective_split(int K, int nsplit) {
    if (nsplit <= 1) return 1;
    int kchunk = ceil_div(ceil_div(K, nsplit), SG_BK) * SG_BK;
    return ceil_div(K, kchunk);
}

}  // namespace crv
