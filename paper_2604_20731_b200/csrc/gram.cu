// gram.cu -- A3: q = G^-1 RES for the Gram matrix of Eq. 26.
//
// G = h^-2 (T (x) I + I (x) T), T = tridiag(-1, 2, -1) of size n = N-1, is a Kronecker SUM,
// so it is diagonalised exactly by the orthonormal DST-I basis S_ia = sqrt(2/N) sin(pi i a/N)
// (S = S^T = S^-1) with eigenvalues h^-2 (lam_a + lam_b), lam_a = 4 sin^2(pi a/(2N)):
//     q = h^2 S [ (S RES S) ./ (lam_a + lam_b) ] S.
// This honours Eq. 28's "factorise once, then substitute" (the factorisation is S and lam,
// built once at create) with an exact transform; the paper's per-axis Thomas argument
// is for the Kronecker-PRODUCT mass matrix and does not apply to G
// (DESIGN.md §5). v1 realises the four n^3 products with the fp32 FFMA GEMM.
#include "common.cuh"
#include "sgemm.cuh"
#include <math.h>

namespace crv {

__global__ void k_gram_constants(float *S, float *lam, int N) {
    int n = N - 1;
    int a = blockIdx.x * blockDim.x + threadIdx.x;
    int i = blockIdx.y;
    if (a >= n) return;
    // sin(pi * i * a / N) with exact integer range reduction: (i*a) mod 2N
    long ia = (long)(i + 1) * (a + 1) % (2L * N);
    double v = sqrt(2.0 / N) * sin(M_PI * (double)ia / (double)N);
    S[(long)i * n + a] = (float)v;
    if (i == 0) {
        double s = sin(M_PI * (double)(a + 1) / (2.0 * N));
        lam[a] = (float)(4.0 * s * s);
    }
}

void gram_init_constants(float *S, float *lam, int N, cudaStream_t s) {
    int n = N - 1;
    dim3 grid(ceil_div(n, 128), n);
    k_gram_constants<<<grid, 128, 0, s>>>(S, lam, N);
}

struct EpiStore {
    float *out;
    int ld;
    float scale;
    __device__ void operator()(int m, int n, float acc, int) const { out[(long)m * ld + n] = acc * scale; }
};

struct EpiEigDiv {
    float *out;
    int ld;
    const float *lam;
    __device__ void operator()(int m, int n, float acc, int) const {
        out[(long)m * ld + n] = acc / (lam[m] + lam[n]);
    }
};

void launch_gram_apply(const float *res, float *q, const float *S, const float *lam, float *w1,
                       float *w2, int N, cudaStream_t s) {
    int n = N - 1;
    float h = 1.0f / (float)N;
    sgemm<false, false>(n, n, n, S, n, res, n, 1, EpiStore{w1, n, 1.0f}, s);        // S R
    sgemm<false, false>(n, n, n, w1, n, S, n, 1, EpiEigDiv{w2, n, lam}, s);         // (S R S) ./ (lam_a+lam_b)
    sgemm<false, false>(n, n, n, S, n, w2, n, 1, EpiStore{w1, n, 1.0f}, s);         // S Z
    sgemm<false, false>(n, n, n, w1, n, S, n, 1, EpiStore{q, n, h * h}, s);         // h^2 S Z S
}

}  // namespace crv
