// mlp_simt.cu -- A1 and A6/A7 with fp32 FFMA (CRVPINN_PREC_FP32): the network
// PINN(x,y) = 16x(1-x)y(1-y) net_theta(x,y) (readings R5/R6) evaluated layer by
// layer over all P = N^2 MLP points (i,j) in [1..N]^2, and its reverse mode.
// Activations are kept in HBM as fp32 [P][w] per hidden layer for the backward pass.
#include "common.cuh"
#include "sgemm.cuh"
#include <math.h>

namespace crv {

static inline int wmax_of(const Net &net) {
    int w = 0;
    for (int l = 1; l < net.nl; ++l) w = net.widths[l] > w ? net.widths[l] : w;
    return w;
}
static inline float *act_ptr(const Net &net, const SimtBufs &b, int a) {
    return b.act + (long)(a - 1) * net.P * wmax_of(net);
}

// ---------------------------------------------------------------- forward
__global__ void k_input_layer(const float *__restrict__ W0, const float *__restrict__ b0,
                              float *__restrict__ act, int N, int w) {
    long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    long P = (long)N * N;
    if (e >= P * w) return;
    int p = (int)(e / w), r = (int)(e % w);
    int i, j;
    point_ij(p, N, i, j);
    float x = (float)i / (float)N, y = (float)j / (float)N;
    act[e] = tanhf(fmaf(W0[2 * r], x, fmaf(W0[2 * r + 1], y, b0[r])));
}

struct EpiTanh {
    float *out;
    int ld;
    const float *bias;
    __device__ void operator()(int m, int n, float acc, int) const {
        out[(long)m * ld + n] = tanhf(acc + bias[n]);
    }
};

// u = cutoff * (W_out t_L + b_out): one warp per point (coalesced over the width).
__global__ void k_output_layer(const float *__restrict__ act, const float *__restrict__ Wo,
                               const float *__restrict__ bo, float *__restrict__ u, int N, int w) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= N * N) return;
    const float *row = act + (long)warp * w;
    float s = 0.0f;
    for (int k = lane; k < w; k += 32) s = fmaf(Wo[k], row[k], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        int i, j;
        point_ij(warp, N, i, j);
        float x = (float)i / (float)N, y = (float)j / (float)N;
        u[(long)j * (N + 1) + i] = cutoff(x, y) * (s + bo[0]);
    }
}

void simt_forward(const Net &net, const float *theta, const SimtBufs &b, float *u, cudaStream_t s) {
    const int N = net.N, P = net.P, nl = net.nl;
    const float *th = theta;
    int w1 = net.widths[1];
    k_input_layer<<<(unsigned)(((long)P * w1 + 255) / 256), 256, 0, s>>>(th + net.woff[0], th + net.boff[0],
                                                                          act_ptr(net, b, 1), N, w1);
    for (int l = 1; l <= nl - 2; ++l) {
        int win = net.widths[l], wout = net.widths[l + 1];
        sgemm<false, true>(P, wout, win, act_ptr(net, b, l), win, th + net.woff[l], win, 1,
                           EpiTanh{act_ptr(net, b, l + 1), wout, th + net.boff[l]}, s);
    }
    int wL = net.widths[nl - 1];
    k_output_layer<<<ceil_div(P * 32, 256), 256, 0, s>>>(act_ptr(net, b, nl - 1), th + net.woff[nl - 1],
                                                          th + net.boff[nl - 1], u, N, wL);
}

int simt_launches_fwd(const Net &net) { return 2 + (net.nl - 2); }

// ---------------------------------------------------------------- continuous evaluation (f1)
// The same network with cutoff at arbitrary points xy[p] = (x, y), p < npts (chunks of at most P
// points, the capacity of the activation buffers).
__global__ void k_input_layer_pts(const float *__restrict__ W0, const float *__restrict__ b0,
                                  float *__restrict__ act, const float *__restrict__ xy, int npts, int w) {
    long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long)npts * w) return;
    int p = (int)(e / w), r = (int)(e % w);
    const float x = xy[2 * (long)p], y = xy[2 * (long)p + 1];
    act[e] = tanhf(fmaf(W0[2 * r], x, fmaf(W0[2 * r + 1], y, b0[r])));
}

__global__ void k_output_layer_pts(const float *__restrict__ act, const float *__restrict__ Wo,
                                   const float *__restrict__ bo, const float *__restrict__ xy,
                                   float *__restrict__ out, int npts, int w) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= npts) return;
    const float *row = act + (long)warp * w;
    float s = 0.0f;
    for (int k = lane; k < w; k += 32) s = fmaf(Wo[k], row[k], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[warp] = cutoff(xy[2 * (long)warp], xy[2 * (long)warp + 1]) * (s + bo[0]);
}

void simt_eval_points(const Net &net, const float *theta, const SimtBufs &b, const float *xy, int npts,
                      float *out, cudaStream_t s) {
    const int nl = net.nl;
    const float *th = theta;
    for (int p0 = 0; p0 < npts; p0 += net.P) {
        const int n = npts - p0 < net.P ? npts - p0 : net.P;
        const float *xyc = xy + 2 * (long)p0;
        int w1 = net.widths[1];
        k_input_layer_pts<<<(unsigned)(((long)n * w1 + 255) / 256), 256, 0, s>>>(th + net.woff[0], th + net.boff[0],
                                                                                act_ptr(net, b, 1), xyc, n, w1);
        for (int l = 1; l <= nl - 2; ++l) {
            int win = net.widths[l], wout = net.widths[l + 1];
            sgemm<false, true>(n, wout, win, act_ptr(net, b, l), win, th + net.woff[l], win, 1,
                               EpiTanh{act_ptr(net, b, l + 1), wout, th + net.boff[l]}, s);
        }
        int wL = net.widths[nl - 1];
        k_output_layer_pts<<<ceil_div(n * 32, 256), 256, 0, s>>>(act_ptr(net, b, nl - 1), th + net.woff[nl - 1],
                                                                  th + net.boff[nl - 1], xyc, out + p0, n, wL);
    }
}

// ---------------------------------------------------------------- backward
// delta_L = gbar * W_out (1 - t_L^2)
__global__ void k_output_bwd(const float *__restrict__ act, const float *__restrict__ Wo,
                             const float *__restrict__ gbar, float *__restrict__ delta, long P, int w) {
    long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P * w) return;
    int p = (int)(e / w), k = (int)(e % w);
    float t = act[e];
    delta[e] = gbar[p] * Wo[k] * (1.0f - t * t);
}

enum { CS_BIAS = 0, CS_FIRST = 1, CS_OUT = 2 };

// Column sums over a chunk of rows: bias gradients, first-layer weight gradients (weights x, y),
// output-layer weight gradients (weight gbar). blockDim.x == w.
template <int MODE>
__global__ void k_colsum(const float *__restrict__ A, int w, int P, int rows_per,
                         const float *__restrict__ gbar, float *__restrict__ partW,
                         float *__restrict__ partB, int N) {
    int c = threadIdx.x, z = blockIdx.x;
    int p0 = z * rows_per, p1 = min(P, p0 + rows_per);
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, sg = 0.0f;
    for (int p = p0; p < p1; ++p) {
        float a = A[(long)p * w + c];
        if (MODE == CS_BIAS) {
            s0 += a;
        } else if (MODE == CS_FIRST) {
            int i, j;
            point_ij(p, N, i, j);
            float x = (float)i / (float)N, y = (float)j / (float)N;
            s0 += a;
            s1 = fmaf(a, x, s1);
            s2 = fmaf(a, y, s2);
        } else {
            float g = gbar[p];
            s1 = fmaf(a, g, s1);
            sg += g;
        }
    }
    if (MODE == CS_BIAS) {
        partB[(long)z * w + c] = s0;
    } else if (MODE == CS_FIRST) {
        partW[(long)z * 2 * w + 2 * c] = s1;
        partW[(long)z * 2 * w + 2 * c + 1] = s2;
        partB[(long)z * w + c] = s0;
    } else {
        partW[(long)z * w + c] = s1;
        if (c == 0) partB[z] = sg;
    }
}

struct EpiPartial {
    float *out;
    long stride;   // floats per split
    int ld;
    __device__ void operator()(int m, int n, float acc, int z) const {
        out[(long)z * stride + (long)m * ld + n] = acc;
    }
};

struct EpiDx {
    float *out;
    int ld;
    const float *tprev;
    __device__ void operator()(int m, int n, float acc, int) const {
        long e = (long)m * ld + n;
        float t = tprev[e];
        out[e] = acc * (1.0f - t * t);
    }
};

void simt_make_plan(const Net &net, MlpPlan &plan) {
    const int P = net.P, nl = net.nl;
    int cs = P / 512;
    if (cs < 1) cs = 1;
    if (cs > 512) cs = 512;
    plan.cs_split = cs;
    plan.rows_per = ceil_div(P, cs);
    plan.cs_split = ceil_div(P, plan.rows_per);
    long off = 0;
    plan.njobs = 0;
    plan.max_count = 0;
    plan.groups = 0;
    auto job = [&](long src, long dst, int count, int nsplit, long stride) {
        RedJob &j = plan.jobs[plan.njobs++];
        j.src = src; j.dst = dst; j.count = count; j.nsplit = nsplit; j.stride = stride;
        j.cols = 1; j.ld = 1; j.transposed = 0; j.scaled = 0;
        if (count > plan.max_count) plan.max_count = count;
    };
    for (int l = 0; l < nl; ++l) {
        int win = net.widths[l], wout = net.widths[l + 1];
        if (l == 0) {
            plan.splitW[l] = plan.cs_split;
            plan.offW[l] = off; off += (long)plan.cs_split * 2 * wout;
            plan.offB[l] = off; off += (long)plan.cs_split * wout;
            job(plan.offW[l], net.woff[l], 2 * wout, plan.cs_split, 2 * wout);
            job(plan.offB[l], net.boff[l], wout, plan.cs_split, wout);
        } else if (l < nl - 1) {
            int tiles = ceil_div(wout, SG_BM) * ceil_div(win, SG_BN);
            int want = ceil_div(600, tiles);
            int maxs = P / 256 > 1 ? P / 256 : 1;
            if (want > maxs) want = maxs;
            plan.splitW[l] = sgemm_effective_split(P, want);
            plan.offW[l] = off; off += (long)plan.splitW[l] * wout * win;
            plan.offB[l] = off; off += (long)plan.cs_split * wout;
            job(plan.offW[l], net.woff[l], wout * win, plan.splitW[l], (long)wout * win);
            job(plan.offB[l], net.boff[l], wout, plan.cs_split, wout);
        } else {
            plan.splitW[l] = plan.cs_split;
            plan.offW[l] = off; off += (long)plan.cs_split * win;
            plan.offB[l] = off; off += (long)plan.cs_split;
            job(plan.offW[l], net.woff[l], win, plan.cs_split, win);
            job(plan.offB[l], net.boff[l], 1, plan.cs_split, 1);
        }
    }
    plan.partial_floats = off;
    plan.groups = reduce_groups(plan.jobs, plan.njobs);
}

void simt_backward(const Net &net, const MlpPlan &plan, const float *theta, const SimtBufs &b,
                   float *grad, cudaStream_t s) {
    const int N = net.N, P = net.P, nl = net.nl;
    const float *th = theta;
    int wL = net.widths[nl - 1];
    float *dcur = b.delta0, *dnext = b.delta1;
    // output layer
    k_output_bwd<<<(unsigned)(((long)P * wL + 255) / 256), 256, 0, s>>>(act_ptr(net, b, nl - 1), th + net.woff[nl - 1],
                                                                        b.gbar, dcur, P, wL);
    k_colsum<CS_OUT><<<plan.cs_split, wL, 0, s>>>(act_ptr(net, b, nl - 1), wL, P, plan.rows_per, b.gbar,
                                                  b.partial + plan.offW[nl - 1], b.partial + plan.offB[nl - 1], N);
    // hidden layers l = nl-2 .. 1: t_{l+1} = tanh(W_l t_l + b_l)
    for (int l = nl - 2; l >= 1; --l) {
        int win = net.widths[l], wout = net.widths[l + 1];
        sgemm<true, false>(wout, win, P, dcur, wout, act_ptr(net, b, l), win, plan.splitW[l],
                           EpiPartial{b.partial + plan.offW[l], (long)wout * win, win}, s);
        k_colsum<CS_BIAS><<<plan.cs_split, wout, 0, s>>>(dcur, wout, P, plan.rows_per, nullptr, nullptr,
                                                         b.partial + plan.offB[l], N);
        sgemm<false, false>(P, win, wout, dcur, wout, th + net.woff[l], win, 1,
                            EpiDx{dnext, win, act_ptr(net, b, l)}, s);
        float *t = dcur; dcur = dnext; dnext = t;
    }
    // first layer: dW0[r][0] = sum delta x, dW0[r][1] = sum delta y, db0 = sum delta
    int w1 = net.widths[1];
    k_colsum<CS_FIRST><<<plan.cs_split, w1, 0, s>>>(dcur, w1, P, plan.rows_per, nullptr,
                                                    b.partial + plan.offW[0], b.partial + plan.offB[0], N);
    launch_reduce(b.partial, grad, b.jobs, plan.njobs, plan.groups, nullptr, s);
}

int simt_launches_bwd(const Net &net) { return 2 + 3 * (net.nl - 2) + 1 + 1; }

}  // namespace crv
