// gram.cu -- A3: q = G^-1 RES for the Gram matrix of Eq. 26.
//
// G = h^-2 (T_x (x) I + I (x) T_y), T = tridiag(-1, 2, -1) of size n = N-1, is a Kronecker SUM.
// The paper's per-axis Thomas shortcut is for the Kronecker-PRODUCT mass
// matrix and is wrong for G. G is solved exactly per axis after a sine
// transform along x:
//   1. R^[j][a] = sum_k RES[j][k] S[k][a]        (DST-I along x, S_ka = sqrt(2/N) sin(pi k a/N))
//   2. for every mode a: (lam_a I + T_y) Z^[:,a] = h^2 R^[:,a],  lam_a = 4 sin^2(pi a/(2N))
//      -- n independent shifted tridiagonal systems along y (batched, one warp each)
//   3. q[j][k] = sum_a Z^[j][a] S[a][k]          (the inverse DST-I along x: S = S^T = S^-1)
// The "factorise once" of Eq. 28 is the per-mode Thomas factor table e[a][j] (built once at
// create, fp64 on the host); every iteration only substitutes. The DSTs are length-2N complex
// FFTs in shared memory (two real rows packed as real/imaginary parts of one complex sequence).
#include "common.cuh"
#include <cmath>
#include <vector>

namespace crv {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// DST-I of two rows per block via a length-M = 2N FFT of the odd extensions packed as
// y = y1 + i y2:  Y = -2i X1 + 2 X2  =>  X1_k = -Im(Y_k)/2, X2_k = Re(Y_k)/2.
// in/out are n x n, addressed (row j, index k) either row-major (j*n+k) or mode-major (k*n+j).
__global__ void k_dst_rows(const float *__restrict__ in, float *__restrict__ out, const float2 *__restrict__ tw,
                           int N, int logM, int in_mode_major, int out_mode_major, float scale) {
    extern __shared__ float2 sa[];
    const int n = N - 1, M = 2 * N;
    const int j0 = 2 * blockIdx.x, j1 = j0 + 1;
    const bool has1 = j1 < n;
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
        int src = -1;
        float sgn = 1.0f;
        if (m >= 1 && m <= n) src = m - 1;
        else if (m > N) { src = M - m - 1; sgn = -1.0f; }
        float v1 = 0.0f, v2 = 0.0f;
        if (src >= 0) {
            if (in_mode_major) {
                v1 = in[(long)src * n + j0];
                if (has1) v2 = in[(long)src * n + j1];
            } else {
                v1 = in[(long)j0 * n + src];
                if (has1) v2 = in[(long)j1 * n + src];
            }
        }
        sa[__brev((unsigned)m) >> (32 - logM)] = make_float2(sgn * v1, sgn * v2);
    }
    __syncthreads();
    for (int lh = 0; lh < logM; ++lh) {
        const int hs = 1 << lh;
        const int tstride = M >> (lh + 1);
        for (int b = threadIdx.x; b < M / 2; b += blockDim.x) {
            const int pos = b & (hs - 1);
            const int i0 = ((b >> lh) << (lh + 1)) + pos, i1 = i0 + hs;
            const float2 w = tw[pos * tstride];
            const float2 u = sa[i0], v = cmul(sa[i1], w);
            sa[i0] = make_float2(u.x + v.x, u.y + v.y);
            sa[i1] = make_float2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
    }
    for (int k = threadIdx.x + 1; k <= n; k += blockDim.x) {
        const float2 Y = sa[k];
        const float x1 = -0.5f * Y.y * scale, x2 = 0.5f * Y.x * scale;
        if (out_mode_major) {
            out[(long)(k - 1) * n + j0] = x1;
            if (has1) out[(long)(k - 1) * n + j1] = x2;
        } else {
            out[(long)j0 * n + (k - 1)] = x1;
            if (has1) out[(long)j1 * n + (k - 1)] = x2;
        }
    }
}

// One warp per mode a: Thomas elimination of (lam_a I + T) z = h2 * r written as two first-order
// linear recurrences (forward g_j = e_{j-1} g_{j-1} + r_j; backward z_j = e_j z_{j+1} + e_j g_j,
// e_j = 1/w_j the precomputed pivots) and evaluated as warp-level affine scans: each lane owns a
// contiguous segment, segment maps are combined with __shfl_up/__shfl_down (Kogge-Stone), then
// every lane replays its segment. Rows are staged in shared memory (odd segment stride: no bank
// conflicts).
constexpr int TRI_WARPS = 4;

__global__ void k_tridiag(const float *__restrict__ rhat, const float *__restrict__ etab, float *__restrict__ z,
                          int n, int seg, float h2) {
    extern __shared__ float sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int a = blockIdx.x * TRI_WARPS + warp;
    if (a >= n) return;
    const int stride = 32 * seg;
    float *sr = sm + (size_t)warp * 2 * stride;   // r, then g, then z
    float *se = sr + stride;
    const float *r = rhat + (size_t)a * n;
    const float *e = etab + (size_t)a * n;
    for (int j = lane; j < n; j += 32) {
        sr[j] = h2 * r[j];
        se[j] = e[j];
    }
    __syncwarp();
    const int j0 = lane * seg, j1 = min(n, j0 + seg);
    // ---- forward: g_j = c_j g_{j-1} + r_j, c_j = e_{j-1} (c_0 = 0)
    float A = 1.0f, B = 0.0f;
    for (int j = j0; j < j1; ++j) {
        const float c = j == 0 ? 0.0f : se[j - 1];
        A = c * A;
        B = c * B + sr[j];
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {   // inclusive scan of maps x -> A x + B
        const float Ap = __shfl_up_sync(0xffffffffu, A, off), Bp = __shfl_up_sync(0xffffffffu, B, off);
        if (lane >= off) { B = A * Bp + B; A = A * Ap; }
    }
    float g = __shfl_up_sync(0xffffffffu, B, 1);
    if (lane == 0) g = 0.0f;
    for (int j = j0; j < j1; ++j) {
        const float c = j == 0 ? 0.0f : se[j - 1];
        g = c * g + sr[j];
        sr[j] = g;
    }
    __syncwarp();
    // ---- backward: z_j = e_j z_{j+1} + e_j g_j (z_n = 0), maps composed from the right
    A = 1.0f;
    B = 0.0f;
    for (int j = j1 - 1; j >= j0; --j) {
        const float ej = se[j];
        A = ej * A;
        B = ej * B + ej * sr[j];
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float Ap = __shfl_down_sync(0xffffffffu, A, off), Bp = __shfl_down_sync(0xffffffffu, B, off);
        if (lane + off < 32) { B = A * Bp + B; A = A * Ap; }
    }
    float zz = __shfl_down_sync(0xffffffffu, B, 1);
    if (lane == 31) zz = 0.0f;
    for (int j = j1 - 1; j >= j0; --j) {
        const float ej = se[j];
        zz = ej * zz + ej * sr[j];
        sr[j] = zz;
    }
    __syncwarp();
    float *zo = z + (size_t)a * n;
    for (int j = lane; j < n; j += 32) zo[j] = sr[j];
}

GramConsts gram_make_constants(int N) {
    GramConsts c{};
    const int n = N - 1, M = 2 * N;
    int logM = 0;
    while ((1 << logM) < M) ++logM;
    c.logM = logM;
    c.seg = (n + 31) / 32;
    if ((c.seg & 1) == 0) c.seg += 1;
    std::vector<float2> tw((size_t)M / 2);
    for (int k = 0; k < M / 2; ++k) {
        const double ang = -2.0 * M_PI * (double)k / (double)M;
        tw[k] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
    std::vector<float> e((size_t)n * n);
    for (int a = 0; a < n; ++a) {
        const double s = std::sin(M_PI * (double)(a + 1) / (2.0 * N));
        const double d = 4.0 * s * s + 2.0;   // lam_a + 2
        double w = d;
        for (int j = 0; j < n; ++j) {
            if (j > 0) w = d - 1.0 / w;
            e[(size_t)a * n + j] = (float)(1.0 / w);
        }
    }
    cudaMalloc(&c.tw, sizeof(float2) * tw.size());
    cudaMalloc(&c.etab, sizeof(float) * e.size());
    cudaMalloc(&c.work, sizeof(float) * 2 * (size_t)n * n);
    cudaMemcpy(c.tw, tw.data(), sizeof(float2) * tw.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(c.etab, e.data(), sizeof(float) * e.size(), cudaMemcpyHostToDevice);
    const int smem_fft = (int)(sizeof(float2) * M);
    const int smem_tri = (int)(sizeof(float) * TRI_WARPS * 2 * 32 * c.seg);
    cudaFuncSetAttribute(k_dst_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_fft);
    cudaFuncSetAttribute(k_tridiag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tri);
    return c;
}

void gram_free_constants(GramConsts &c) {
    cudaFree(c.tw);
    cudaFree(c.etab);
    cudaFree(c.work);
    c = GramConsts{};
}

void launch_gram_apply(const float *res, float *q, const GramConsts &c, int N, cudaStream_t s) {
    const int n = N - 1, M = 2 * N;
    const float h = 1.0f / (float)N;
    const float nrm = sqrtf(2.0f / (float)N);
    float *rhat = c.work, *zhat = c.work + (size_t)n * n;
    const int fft_threads = M / 2 < 512 ? M / 2 : 512;
    const int rows = (n + 1) / 2;
    k_dst_rows<<<rows, fft_threads, sizeof(float2) * M, s>>>(res, rhat, c.tw, N, c.logM, 0, 1, nrm);
    k_tridiag<<<ceil_div(n, TRI_WARPS), 32 * TRI_WARPS, sizeof(float) * TRI_WARPS * 2 * 32 * c.seg, s>>>(
        rhat, c.etab, zhat, n, c.seg, h * h);
    k_dst_rows<<<rows, fft_threads, sizeof(float2) * M, s>>>(zhat, q, c.tw, N, c.logM, 1, 0, nrm);
}

}  // namespace crv
