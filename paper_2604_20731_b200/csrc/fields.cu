// fields.cu -- lattice kernels of the CRVPINN update on sm_100a: A0 setup, A7 partial
// reduction, A8 Adam.
// HBM-bound elementwise / stencil work: coalesced along x (i), one pass per field.
#include "common.cuh"
#include <math.h>

namespace crv {


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

// b = h^2 f_total, f_total = f - div+(g K beta) (reading R1: f_total is the right side of
// -div(alpha grad p) = f_total; Eq. 23's RHS with the sign of R1). The gravity term (PAPER.md:370,
// reading R23): g = -Gr y-hat, beta = (1-S) + M r S (r = rho_g/rho_w), so with gamma = K beta
// -div+(g gamma)_{i,j} = Gr (gamma_{i,j+1} - gamma_{i,j}) / h (Eq. 22's forward difference in y).
__device__ __forceinline__ float gamma_node(const float *K, const float *S, long p, float Mr) {
    const float s = fminf(fmaxf(S[p], 0.0f), 1.0f);
    return K[p] * ((1.0f - s) + Mr * s);
}

__global__ void k_rhs(const float *__restrict__ K, const float *__restrict__ S, const float *__restrict__ f,
                      float *__restrict__ b, int N, float h, float Mr, float Gr) {
    const long nn = (long)(N + 1) * (N + 1);
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nn) return;
    float v = h * h * f[p];
    const int j = (int)(p / (N + 1));
    if (Gr != 0.0f && j < N) v += h * Gr * (gamma_node(K, S, p + N + 1, Mr) - gamma_node(K, S, p, Mr));
    b[p] = v;
}

void launch_rhs(const float *K, const float *S, const float *f, float *b, int N, float mobility, float rho_ratio,
                float gravity, cudaStream_t s) {
    long nn = (long)(N + 1) * (N + 1);
    k_rhs<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(K, S, f, b, N, 1.0f / (float)N, mobility * rho_ratio, gravity);
}

// A2-A5 (residual, Gram solve, loss, adjoint) live in gram.cu as one fused chain.

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
                                                        const DevState *st, AdamOp A) {
    __shared__ float sh[RED_WARPS][33];
    pdl_wait();
    pdl_trigger();
    // the Adam step counter: one writer (bc1/bc2 of this step were set by the field chain)
    if (A.on && blockIdx.x == 0 && threadIdx.x == 0 && !A.st->nonfinite) A.st->t = A.st->t + 1;
    int j = 0, g = blockIdx.x;
    while (j < njobs && g >= red_groups(jobs[j])) { g -= red_groups(jobs[j]); ++j; }
    if (j >= njobs) return;
    const RedJob jb = jobs[j];
    const float sc = red_scale(jb, st);
    if (red_wide(jb)) {
        const int o = g * RED_THREADS + threadIdx.x;
        if (o >= jb.count) return;
        const AdamPre ap = A.on ? adam_pre(A, jb.dst + o) : AdamPre{};
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
        if (A.on) adam_one(A, jb.dst + o, s * sc, ap);
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int o = g * 32 + lane;
    const AdamPre ap = (A.on && warp == 0 && o < jb.count) ? adam_pre(A, jb.dst + o) : AdamPre{};
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
        if (A.on) adam_one(A, jb.dst + o, t * sc, ap);
    }
}

// One hidden-layer weight job (transposed == 2 layout with cols == ld, count % 4 == 0) with small
// blocks and no shared memory: a 64-thread CTA fits next to a k_tc_bwd2 CTA (which leaves ~11K
// registers and ~1.5 KB of shared memory per SM), so the reduction of GEMM g's dW partials runs on
// a side stream underneath the backward of GEMM g-1 instead of after the last one. A warp owns four
// consecutive float4 outputs (lane & 3) and splits their sums over eight lane groups (lane >> 2:
// splits sg, sg + 8, ...), all loads of a lane in flight together; the eight group sums are combined
// by a fixed butterfly and lane group 0 keeps the result: the order depends only on nsplit.
constexpr int RW_THREADS = 64;
__global__ void __launch_bounds__(RW_THREADS) k_reduce_wide(const float *__restrict__ partial,
                                                            float *__restrict__ grad, RedJobSet js,
                                                            const DevState *st, AdamOp A) {
    const RedJob jb = js.j[blockIdx.y];   // one job per grid row: the jobs of a launch run concurrently
    const float sc = red_scale(jb, st);
    const int n4 = jb.count >> 2;
    const int lane = threadIdx.x & 31, og = lane & 3, sg = lane >> 2;
    const int wpb = RW_THREADS / 32;
    const long st4 = jb.stride >> 2;
    for (int q0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * 4; q0 < n4; q0 += gridDim.x * wpb * 4) {
        const int q = q0 + og;
        // lane (og, sg < 4) finishes component sg of output float4 og: its Adam state first
        const AdamPre ap = (A.on && sg < 4 && q < n4) ? adam_pre(A, jb.dst + 4 * (long)q + (sg & 3)) : AdamPre{};
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < n4) {
            const float4 *src = reinterpret_cast<const float4 *>(partial + jb.src + red_off(jb, 4 * q));
            int z = sg;
            for (; z + 56 < jb.nsplit; z += 64) {   // eight loads in flight per lane
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (long)(z + 8 * u) * st4);
#pragma unroll
                for (int u = 0; u < 8; ++u) { s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w; }
            }
            for (; z + 24 < jb.nsplit; z += 32) {
                float4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(src + (long)(z + 8 * u) * st4);
#pragma unroll
                for (int u = 0; u < 4; ++u) { s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w; }
            }
            for (; z < jb.nsplit; z += 8) {
                const float4 v = __ldg(src + (long)z * st4);
                s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
            }
        }
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
            s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
            s.z += __shfl_xor_sync(0xffffffffu, s.z, off);
            s.w += __shfl_xor_sync(0xffffffffu, s.w, off);
        }
        // lane group 0's sums (one summation order) to lanes (og, sg < 4): lane (og, k) finishes
        // component k of output float4 og -- 16 lanes share the gradient stores and the Adam updates
        const int k = sg & 3;
        const float c0 = __shfl_sync(0xffffffffu, s.x, og), c1 = __shfl_sync(0xffffffffu, s.y, og);
        const float c2 = __shfl_sync(0xffffffffu, s.z, og), c3 = __shfl_sync(0xffffffffu, s.w, og);
        if (sg < 4 && q < n4) {
            const float r = (k == 0 ? c0 : k == 1 ? c1 : k == 2 ? c2 : c3) * sc;
            const long d = jb.dst + 4 * (long)q + k;
            grad[d] = r;
            if (A.on) adam_one(A, d, r, ap);
        }
    }
}

// The same reduction, one thread per float4 output summing all splits in order (8 loads in flight):
// more outputs per warp in flight, for the launches that run on one CTA per SM beside a backward GEMM
__global__ void __launch_bounds__(RW_THREADS) k_reduce_wide_seq(const float *__restrict__ partial,
                                                                float *__restrict__ grad, RedJob jb,
                                                                const DevState *st, AdamOp A) {
    const float sc = red_scale(jb, st);
    const int n4 = jb.count >> 2;
    for (int q = blockIdx.x * RW_THREADS + threadIdx.x; q < n4; q += gridDim.x * RW_THREADS) {
        const float4 *src = reinterpret_cast<const float4 *>(partial + jb.src + red_off(jb, 4 * q));
        const long st4 = jb.stride >> 2;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        int z = 0;
        for (; z + 8 <= jb.nsplit; z += 8) {
            float4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(src + (long)(z + k) * st4);
#pragma unroll
            for (int k = 0; k < 8; ++k) { s.x += v[k].x; s.y += v[k].y; s.z += v[k].z; s.w += v[k].w; }
        }
        for (; z < jb.nsplit; ++z) {
            const float4 v = __ldg(src + (long)z * st4);
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
        float *d = grad + jb.dst + 4 * q;   // dst offsets are not 16-byte aligned in theta
        d[0] = s.x * sc; d[1] = s.y * sc; d[2] = s.z * sc; d[3] = s.w * sc;
        if (A.on) {
            const long e = jb.dst + 4 * (long)q;
            adam_one(A, e, s.x * sc);
            adam_one(A, e + 1, s.y * sc);
            adam_one(A, e + 2, s.z * sc);
            adam_one(A, e + 3, s.w * sc);
        }
    }
}

void launch_reduce_wide(const float *partial, float *grad, const RedJob &job, const DevState *st, int max_ctas,
                        cudaStream_t s, const AdamOp *A) {
    AdamOp a{};
    if (A) a = *A;
    if (max_ctas < 0) {   // beside a GEMM: one CTA per SM
        k_reduce_wide_seq<<<-max_ctas, RW_THREADS, 0, s>>>(partial, grad, job, st, a);
        return;
    }
    RedJobSet js{};
    js.j[0] = job;
    js.n = 1;
    launch_reduce_wide_set(partial, grad, js, st, max_ctas, s, A);
}

void launch_reduce_wide_set(const float *partial, float *grad, const RedJobSet &js, const DevState *st,
                            int max_ctas, cudaStream_t s, const AdamOp *A) {
    if (js.n < 1) return;
    AdamOp a{};
    if (A) a = *A;
    int n4 = 0;
    for (int k = 0; k < js.n; ++k) n4 = js.j[k].count / 4 > n4 ? js.j[k].count / 4 : n4;
    int grid = (n4 + 4 * (RW_THREADS / 32) - 1) / (4 * (RW_THREADS / 32));
    if (grid * js.n > max_ctas) grid = max_ctas / js.n;
    if (grid < 1) grid = 1;
    k_reduce_wide<<<dim3(grid, js.n), RW_THREADS, 0, s>>>(partial, grad, js, st, a);
}

int reduce_groups(const RedJob *jobs, int njobs) {
    int gsum = 0;
    for (int j = 0; j < njobs; ++j) gsum += red_groups(jobs[j]);
    return gsum;
}

void launch_reduce(const float *partial, float *grad, const RedJob *jobs, int njobs, int total_groups,
                   const DevState *st, cudaStream_t s, const AdamOp *A) {
    AdamOp a{};
    if (A) a = *A;
    launch_pdl(k_reduce, dim3(total_groups), dim3(RED_THREADS), 0, s, 1, partial, grad, jobs, njobs, st, a);
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

// A8 with an AdamOp over a whole gradient vector (tensor path with a gradient exchange: the update
// must follow the all-reduce, so it cannot ride on the reductions)
__global__ void k_adam_op(const float *__restrict__ g, long np, AdamOp A) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    pdl_wait();
    pdl_trigger();
    if (e == 0 && !A.st->nonfinite) A.st->t = A.st->t + 1;
    if (e < np) adam_one(A, e, g[e]);
}

void launch_adam_op(const float *g, long np, const AdamOp &A, cudaStream_t s) {
    launch_pdl(k_adam_op, dim3((unsigned)((np + 255) / 256)), dim3(256), 0, s, 1, g, np, A);
}

__global__ void k_begin_call(DevState *st) {
    st->it = 0;
    st->nonfinite = 0;
}

void launch_begin_call(DevState *st, cudaStream_t s) { k_begin_call<<<1, 1, 0, s>>>(st); }

}  // namespace crv
