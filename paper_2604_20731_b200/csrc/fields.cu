// fields.cu -- lattice kernels of the CRVPINN update on sm_100a: A0 setup, A2 residual
// stencil, A4 loss reduction, A5 adjoint stencil, A7 partial reduction, A8 Adam.
// HBM-bound elementwise / stencil work: coalesced along x (i), one pass per field.
#include "common.cuh"
#include <math.h>

namespace crv {

__device__ __forceinline__ long lat(int i, int j, int N) { return (long)j * (N + 1) + i; }

// ---------------------------------------------------------------- A0 (reading R10)
__global__ void k_alpha(const float *__restrict__ K, const float *__restrict__ S,
                        float *__restrict__ alpha, long nn, float M) {
    long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nn) return;
    float s = fminf(fmaxf(S[p], 0.0f), 1.0f);
    alpha[p] = K[p] * ((1.0f - s) + M * s);
}

void launch_alpha(const float *K, const float *S, float *alpha, int N, float mobility, cudaStream_t s) {
    long nn = (long)(N + 1) * (N + 1);
    k_alpha<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(K, S, alpha, nn, mobility);
}

// b = h^2 f (reading R1: f is the right side of -div(alpha grad p) = f)
__global__ void k_scale_b(const float *__restrict__ f, float *__restrict__ b, long nn, float h2) {
    long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < nn) b[p] = h2 * f[p];
}

void launch_scale_b(const float *f, float *b, int N, cudaStream_t s) {
    long nn = (long)(N + 1) * (N + 1);
    float h = 1.0f / (float)N;
    k_scale_b<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(f, b, nn, h * h);
}

// ---------------------------------------------------------------- A2: residual (Eq. 25)
// RES_kl = a_{k-1,l}(u_kl-u_{k-1,l}) + a_{k,l-1}(u_kl-u_{k,l-1}) + a_kl(2u_kl-u_{k+1,l}-u_{k,l+1}) - b_kl,
// the closed form of (alpha grad+ u, grad+ delta_kl)_h - (RHS, delta_kl)_h (reading R16: the
// x-edge (k-1,l)->(k,l) carries alpha of its tail node, as grad+ places it).
__global__ void k_residual(const float *__restrict__ u, const float *__restrict__ alpha,
                           const float *__restrict__ b, float *__restrict__ res, int N) {
    int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
    int l = blockIdx.y + 1;
    int n = N - 1;
    if (k > n) return;
    float uc = u[lat(k, l, N)];
    float r = alpha[lat(k - 1, l, N)] * (uc - u[lat(k - 1, l, N)])
            + alpha[lat(k, l - 1, N)] * (uc - u[lat(k, l - 1, N)])
            + alpha[lat(k, l, N)] * ((uc - u[lat(k + 1, l, N)]) + (uc - u[lat(k, l + 1, N)]))
            - b[lat(k, l, N)];
    res[(long)(l - 1) * n + (k - 1)] = r;
}

void launch_residual(const float *u, const float *alpha, const float *b, float *res, int N, cudaStream_t s) {
    int n = N - 1;
    dim3 grid(ceil_div(n, 128), n);
    k_residual<<<grid, 128, 0, s>>>(u, alpha, b, res, N);
}

// ---------------------------------------------------------------- A4: LOSS = RES^T q (Eq. 27)
// fp32 products, fp64 accumulation, fixed-order block + final reductions (deterministic).
int loss_partial_blocks(int n2) {
    int b = ceil_div(n2, 2048);
    return b < 1 ? 1 : (b > 296 ? 296 : b);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void k_loss_partials(const float *__restrict__ res, const float *__restrict__ q,
                                double *__restrict__ part, int n2) {
    __shared__ double sh[8];
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += gridDim.x * blockDim.x)
        acc += (double)(res[i] * q[i]);
    acc = warp_sum_d(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sh[w];
        part[blockIdx.x] = s;
    }
}

void launch_loss_partials(const float *res, const float *q, double *part, int n2, int nblk, cudaStream_t s) {
    k_loss_partials<<<nblk, 256, 0, s>>>(res, q, part, n2);
}

// Final sum + bookkeeping: history slot, non-finite flag, Adam bias corrections for step t+1.
__global__ void k_loss_final(const double *__restrict__ part, int nblk, DevState *st,
                             double *hist, int n_hist, double beta1, double beta2, int advance) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nblk; i += 256) acc += part[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double loss = sh[0];
        st->loss = loss;
        st->gmax_bits = 0u;
        if (hist != nullptr && st->it < n_hist) hist[st->it] = loss;
        st->it += 1;
        if (!isfinite(loss)) st->nonfinite = 1;
        if (advance && !st->nonfinite) {
            int64_t t = st->t + 1;
            st->bc1 = 1.0 - pow(beta1, (double)t);
            st->bc2 = 1.0 - pow(beta2, (double)t);
        }
    }
}

void launch_loss_final(const double *part, int nblk, DevState *st, double *hist, int n_hist,
                       double beta1, double beta2, cudaStream_t s) {
    // beta1 < 0 encodes "evaluation only" (no Adam step follows)
    int advance = beta1 >= 0.0;
    k_loss_final<<<1, 256, 0, s>>>(part, nblk, st, hist, n_hist, advance ? beta1 : 0.9,
                                   advance ? beta2 : 0.999, advance);
}

// ---------------------------------------------------------------- A5: adjoint
// g_u = dLOSS/du = 2 A(alpha) q (A symmetric: the same stencil on q, q = 0 off the interior),
// then gbar_p = g_u * cutoff(x_p, y_p) (chain rule through u = cutoff * net) at every MLP point
// p = (i,j) in [1..N]^2 (zero on the boundary rows i = N or j = N). With track_max the block
// maxima of |gbar| are folded into DevState::gmax_bits (order-independent, deterministic).
__global__ void k_adjoint(const float *__restrict__ q, const float *__restrict__ alpha,
                          float *__restrict__ gbar, float *__restrict__ gu_lat, int N,
                          DevState *st, int track_max) {
    __shared__ float smax[8];
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    float g = 0.0f, gb = 0.0f;
    int n = N - 1;
    if (p < N * N) {
        int i, j;
        point_ij(p, N, i, j);
        if (i <= n && j <= n) {
            auto Q = [&](int a, int c) -> float {
                return (a >= 1 && a <= n && c >= 1 && c <= n) ? q[(long)(c - 1) * n + (a - 1)] : 0.0f;
            };
            float qc = Q(i, j);
            float aq = alpha[lat(i - 1, j, N)] * (qc - Q(i - 1, j))
                     + alpha[lat(i, j - 1, N)] * (qc - Q(i, j - 1))
                     + alpha[lat(i, j, N)] * ((qc - Q(i + 1, j)) + (qc - Q(i, j + 1)));
            g = 2.0f * aq;
            float x = (float)i / (float)N, y = (float)j / (float)N;
            gb = g * cutoff(x, y);
        }
        gbar[p] = gb;
        if (gu_lat) gu_lat[lat(i, j, N)] = g;
    }
    if (track_max) {
        float m = fabsf(gb);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; ++w) m = fmaxf(m, smax[w]);
            if (m > 0.0f) atomicMax(&st->gmax_bits, __float_as_uint(m));
        }
    }
}

void launch_adjoint(const float *q, const float *alpha, float *gbar, float *gu_lattice, int N,
                    DevState *st, int track_max, cudaStream_t s) {
    int P = N * N;
    k_adjoint<<<ceil_div(P, 256), 256, 0, s>>>(q, alpha, gbar, gu_lattice, N, st, track_max);
}

// ---------------------------------------------------------------- A7: deterministic reduction
// Blocks of 1024 threads. A job with few splits (nsplit <= 64) or many outputs (the weight-gradient
// GEMM partials) is "wide": one thread per output, 8 independent loads in flight, summed in split order. A job
// with many splits and few outputs (column-sum partials of the per-CTA kernels) is "deep": one
// block per 32 outputs, warp w sums splits w, w+32, ..., then the 32 warp sums are added in warp
// order. Either way the order depends only on (nsplit, output): deterministic.
constexpr int RED_THREADS = 1024;
constexpr int RED_WARPS = RED_THREADS / 32;

// wide: few splits, or enough outputs to fill the GPU with one thread per output
__host__ __device__ inline bool red_wide(const RedJob &j) { return j.nsplit <= 64 || j.count >= 8192; }

__host__ __device__ inline int red_groups(const RedJob &j) {
    return red_wide(j) ? (j.count + RED_THREADS - 1) / RED_THREADS : (j.count + 31) / 32;
}

__device__ __forceinline__ long red_off(const RedJob &jb, int o) {
    return jb.transposed == 1 ? (long)(o % jb.cols) * jb.ld + (o / jb.cols)
         : jb.transposed == 2 ? (long)(o / jb.cols) * jb.ld + (o % jb.cols) : (long)o;
}

__global__ void __launch_bounds__(RED_THREADS) k_reduce(const float *__restrict__ partial, float *__restrict__ grad,
                                                        const RedJob *__restrict__ jobs, int njobs,
                                                        const DevState *st) {
    __shared__ float sh[RED_WARPS][33];
    int j = 0, g = blockIdx.x;
    while (j < njobs && g >= red_groups(jobs[j])) { g -= red_groups(jobs[j]); ++j; }
    if (j >= njobs) return;
    const RedJob jb = jobs[j];
    const float sc = jb.scaled ? st->inv_gscale : 1.0f;
    if (red_wide(jb)) {
        const int o = g * RED_THREADS + threadIdx.x;
        if (o >= jb.count) return;
        const float *src = partial + jb.src + red_off(jb, o);
        float s = 0.0f;
        int z = 0;
        for (; z + 8 <= jb.nsplit; z += 8) {
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(src + (long)(z + k) * jb.stride);
#pragma unroll
            for (int k = 0; k < 8; ++k) s += v[k];
        }
        for (; z < jb.nsplit; ++z) s += __ldg(src + (long)z * jb.stride);
        grad[jb.dst + o] = s * sc;
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int o = g * 32 + lane;
    float s = 0.0f;
    if (o < jb.count) {
        const float *src = partial + jb.src + red_off(jb, o);
        int z = warp;
        for (; z + 3 * RED_WARPS < jb.nsplit; z += 4 * RED_WARPS) {
            const float v0 = __ldg(src + (long)z * jb.stride);
            const float v1 = __ldg(src + (long)(z + RED_WARPS) * jb.stride);
            const float v2 = __ldg(src + (long)(z + 2 * RED_WARPS) * jb.stride);
            const float v3 = __ldg(src + (long)(z + 3 * RED_WARPS) * jb.stride);
            s += v0; s += v1; s += v2; s += v3;
        }
        for (; z < jb.nsplit; z += RED_WARPS) s += __ldg(src + (long)z * jb.stride);
    }
    sh[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && o < jb.count) {
        float t = 0.0f;
        for (int w = 0; w < RED_WARPS; ++w) t += sh[w][lane];
        grad[jb.dst + o] = t * sc;
    }
}

int reduce_groups(const RedJob *jobs, int njobs) {
    int gsum = 0;
    for (int j = 0; j < njobs; ++j) gsum += red_groups(jobs[j]);
    return gsum;
}

void launch_reduce(const float *partial, float *grad, const RedJob *jobs, int njobs, int total_groups,
                   const DevState *st, cudaStream_t s) {
    k_reduce<<<total_groups, RED_THREADS, 0, s>>>(partial, grad, jobs, njobs, st);
}

// ---------------------------------------------------------------- A8: Adam
__global__ void k_adam(float *__restrict__ theta, float *__restrict__ m, float *__restrict__ v,
                       const float *__restrict__ g, long np, const DevState *st,
                       DevState *st_w, float lr, float beta1, float beta2, float eps) {
    long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (st->nonfinite) return;
    float bc1 = (float)st->bc1, bc2 = (float)st->bc2;
    if (k == 0) st_w->t = st->t + 1;   // the only writer of t; other blocks read bc1/bc2 only
    if (k >= np) return;
    float gk = g[k];
    if (!isfinite(gk)) {
        atomicExch(&st_w->nonfinite, 1);
        return;
    }
    float mk = beta1 * m[k] + (1.0f - beta1) * gk;
    float vk = beta2 * v[k] + (1.0f - beta2) * gk * gk;
    m[k] = mk;
    v[k] = vk;
    float mh = mk / bc1, vh = vk / bc2;
    theta[k] -= lr * mh / (sqrtf(vh) + eps);
}

void launch_adam(float *theta, float *m, float *v, const float *g, long np, const DevState *st,
                 DevState *st_w, float lr, float beta1, float beta2, float eps, cudaStream_t s) {
    k_adam<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(theta, m, v, g, np, st, st_w, lr, beta1, beta2, eps);
}

__global__ void k_begin_call(DevState *st) {
    st->it = 0;
    st->nonfinite = 0;
}

void launch_begin_call(DevState *st, cudaStream_t s) { k_begin_call<<<1, 1, 0, s>>>(st); }

}  // namespace crv
