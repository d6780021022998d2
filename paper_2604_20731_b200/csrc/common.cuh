// common.cuh -- shared device/host definitions of the CRVPINN sm_100a library.
// Product code only: nothing here is shared with oracle/ (DESIGN.md §1).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

#define CRV_MAX_LAYERS 16

namespace crv {

// Device-resident per-context scalars. One instance lives in device memory.
struct DevState {
    double loss;          // LOSS of the last evaluated iteration (Eq. 27)
    double bc1, bc2;      // Adam bias corrections 1-beta^t for the pending update
    int64_t t;            // Adam step counter (persists across calls, reading R8)
    int it;               // index into the loss history for the current call
    int nonfinite;        // set when a non-finite loss / gradient is seen
    float gscale;         // power-of-two scale applied to dLOSS/dnet in the tensor backward
    float inv_gscale;
    unsigned gmax_bits;   // max |dLOSS/dnet| of the current iteration (float bits, atomicMax)
    int pad;
    // Tensor path, per hidden GEMM g: the fp16 weight copies hold W_g 2^-wexp[g]
    // (max |.| <= 2^14 for the whole call), and the backward stores Delta one level down with an extra
    // factor 2^-fexp[g] (fexp = round(log2(|W_g|_F / sqrt(fan_in))), 0 for Xavier-scaled weights), so
    // fp16 holds weights and Delta of any magnitude. Set per call by k_wscale.
    int wexp[CRV_MAX_LAYERS];
    int fexp[CRV_MAX_LAYERS];
};

// Geometry and network description passed by value to kernels.
struct Net {
    int N;                // grid intervals; MLP points are (i,j) in [1..N]^2 -> P = N*N
    int n;                // N-1 interior nodes per axis
    int P;                // N*N MLP points
    int nl;               // weight layers (hidden + output)
    int widths[CRV_MAX_LAYERS + 1];
    long woff[CRV_MAX_LAYERS];
    long boff[CRV_MAX_LAYERS];
};

// Job of the deterministic partial-sum reducer: dst[o] = scale * sum_{z<nsplit} src[z*stride + off(o)],
// o < count, off(o) = o (transposed = 0), (o % cols) * ld + o / cols (1), (o / cols) * ld + o % cols (2).
struct RedJob {
    long src;      // offset in the partial buffer
    long dst;      // offset in the gradient vector
    long stride;   // floats between consecutive splits
    int count;
    int nsplit;
    int cols, ld;  // transposed layout parameters
    int transposed;
    int scaled;    // tensor backward partials: multiply by DevState::inv_gscale x 2^(sum_{g_lo <= g < g_hi}
                   // fexp[g] - 14 tsc) (the Delta level's cumulative scale; tsc: the partials carry one
                   // activation factor t' = 2^14 t)
    int g_lo, g_hi, tsc;
};

// several reduction jobs in one launch (kernel parameter)
struct RedJobSet {
    RedJob j[CRV_MAX_LAYERS];
    int n;
};

// unscale factor of a reduction job (RedJob::scaled)
__device__ __forceinline__ float red_scale(const RedJob &j, const DevState *st) {
    if (!j.scaled) return 1.0f;
    int e = j.tsc ? -14 : 0;
    for (int g = j.g_lo; g < j.g_hi; ++g) e += st->fexp[g];
    return st->inv_gscale * exp2f((float)e);
}

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// A8 (Adam; reading R7) fused into the weight-gradient reductions of the tensor path:
// the thread that finishes gradient entry e updates theta[e], m[e], v[e] and the tensor path's
// operand copies of that parameter. on = 0: the reductions only write the gradient (loss_grad, the
// fp32 path, whose Adam is k_adam).
struct AdamOp {
    int on;
    float *theta, *m, *v;
    DevState *st;
    float lr, beta1, beta2, eps;
    Net net;
    int WP, KC;
    __half *Wf, *WTf;                 // hidden weights, fp16, 2^-wexp scaled, B-operand block layouts
    float *W1p, *bp, *Wop;            // first layer / biases (x 2 log2 e) and output layer, fp32
};

constexpr float ADAM_TANH_C = 2.8853900817779268f;   // 2 log2(e) (the forward's pre-scale of W1 and biases)

// Adam state of entry e, loaded ahead of the gradient it will be combined with (the reductions issue
// these loads before their partial-sum loads, so the two latencies overlap)
struct AdamPre {
    float m, v, th;
};
__device__ __forceinline__ AdamPre adam_pre(const AdamOp &A, long e) { return {A.m[e], A.v[e], A.theta[e]}; }

__device__ __forceinline__ void adam_one(const AdamOp &A, long e, float gk, const AdamPre &p) {
    DevState *st = A.st;
    if (st->nonfinite) return;
    if (!isfinite(gk)) {
        atomicExch(&st->nonfinite, 1);
        return;
    }
    const float bc1 = (float)st->bc1, bc2 = (float)st->bc2;
    const float mk = A.beta1 * p.m + (1.0f - A.beta1) * gk;
    const float vk = A.beta2 * p.v + (1.0f - A.beta2) * gk * gk;
    A.m[e] = mk;
    A.v[e] = vk;
    const float th = p.th - A.lr * (mk / bc1) / (sqrtf(vk / bc2) + A.eps);
    A.theta[e] = th;
    const Net &net = A.net;
    const int nl = net.nl, L = nl - 1, WP = A.WP, KC = A.KC;
    int l = 0;
    while (l + 1 < nl && e >= net.woff[l + 1]) ++l;
    const int win = net.widths[l];
    if (e >= net.boff[l]) {   // bias of layer l
        const int o = (int)(e - net.boff[l]);
        if (l < L) A.bp[l * WP + o] = ADAM_TANH_C * th;
        else A.Wop[WP] = th;
        return;
    }
    const long r = e - net.woff[l];
    const int o = (int)(r / win), i = (int)(r % win);   // W_l[o][i]
    if (l == 0) {
        A.W1p[2 * o + i] = ADAM_TANH_C * th;
    } else if (l == L) {
        A.Wop[i] = th;
    } else {
        const int gg = l - 1;
        const __half hv = __float2half_rn(ldexpf(th, -st->wexp[gg]));
        {   // Wf: row n = o, K index k = i
            const size_t blk = ((size_t)gg * KC + (i >> 6)) * (size_t)WP * 64;
            A.Wf[blk + (uint32_t)(o * 64 + ((((i & 63) >> 3) ^ (o & 7)) << 3) + (i & 7))] = hv;
        }
        {   // WTf: row n = i, K index k = o
            const size_t blk = ((size_t)gg * KC + (o >> 6)) * (size_t)WP * 64;
            A.WTf[blk + (uint32_t)(i * 64 + ((((o & 63) >> 3) ^ (i & 7)) << 3) + (o & 7))] = hv;
        }
    }
}

__device__ __forceinline__ void adam_one(const AdamOp &A, long e, float gk) { adam_one(A, e, gk, adam_pre(A, e)); }

// Programmatic dependent launch (PDL): kernels of the iteration are launched with programmatic
// stream serialization, so a kernel's CTAs may start (prologue: barrier init, TMEM alloc) while the
// previous kernel drains; pdl_wait() blocks until the previous grid has completed and its memory
// is visible, pdl_trigger() lets the next grid be scheduled as soon as SMs free up.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              int cluster_x, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (cluster_x > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster_x;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}

// MLP point p -> lattice node (i, j) in [1..N]^2
__device__ __forceinline__ void point_ij(int p, int N, int &i, int &j) {
    i = (p & (N - 1)) + 1;   // N is a power of two
    j = (p / N) + 1;
}

__device__ __forceinline__ float cutoff(float x, float y) {
    return 16.0f * x * (1.0f - x) * y * (1.0f - y);
}

}  // namespace crv

// ------------------------------------------------------------------ launch wrappers
// (defined in the .cu files; all take the context stream)
namespace crv {
// fields.cu
void launch_alpha(const float *K, const float *S, float *alpha, int N, float mobility, cudaStream_t s);
void launch_rhs(const float *K, const float *S, const float *f, float *b, int N, float mobility, float rho_ratio,
                float gravity, cudaStream_t s);
void launch_adam(float *theta, float *m, float *v, const float *g, long np, const DevState *st,
                 DevState *st_w, float lr, float beta1, float beta2, float eps, cudaStream_t s);
void launch_begin_call(DevState *st, cudaStream_t s);
void launch_adam_op(const float *g, long np, const AdamOp &A, cudaStream_t s);
// total_groups = reduce_groups(host copy of jobs)
int reduce_groups(const RedJob *jobs, int njobs);
// A = nullptr or A->on == 0: gradient only; max_ctas: grid cap of the split-group kernel (launches
// with the SMs to themselves); -n: n CTAs of the one-thread-per-output kernel (beside a GEMM)
void launch_reduce_wide(const float *partial, float *grad, const RedJob &job, const DevState *st, int max_ctas,
                        cudaStream_t s, const AdamOp *A = nullptr);
void launch_reduce(const float *partial, float *grad, const RedJob *jobs, int njobs, int total_groups,
                   const DevState *st, cudaStream_t s, const AdamOp *A = nullptr);
// the split-group kernel over several jobs at once (grid rows = jobs), up to max_ctas CTAs in all
void launch_reduce_wide_set(const float *partial, float *grad, const RedJobSet &js, const DevState *st,
                            int max_ctas, cudaStream_t s, const AdamOp *A = nullptr);
// gram.cu
struct GramConsts {
    float2 *tw = nullptr;   // FFT twiddles per stage: [hs + pos] = exp(-2 pi i pos / 2hs), 2N entries
    float *etab = nullptr;  // per-mode Thomas pivots 1/w_j, mode-major [a][j]
    float *work = nullptr;  // 2 n^2 scratch (R^, Z^)
    int logM = 0, seg = 0;
    void *pcg = nullptr;    // f2 workspace (vectors, CG state, the two-iteration graph), made on first use
};
GramConsts gram_make_constants(int N);
void gram_free_constants(GramConsts &c);
// A2-A5 fused: residual + DST, tridiagonal solves, inverse DST + loss partials, adjoint + loss
int field_chain_loss_blocks(int N);
void launch_field_chain(const float *u, const float *alpha, const float *b, float *res, float *q, float *gbar,
                        float *gu_lat, double *loss_part, const GramConsts &c, int N, DevState *st, int track_max,
                        double *hist, int n_hist, double beta1, double beta2, int advance, cudaStream_t s);
// f2: A(alpha) u = b by Gram-preconditioned CG (u_lat: interior written, boundary untouched);
// returns 0 / -1 (CUDA error); iterations used and the final true relative residual
int pcg_solve(const float *alpha, const float *b, float *u_lat, GramConsts &c, int N, double rtol, int max_iter,
              int *iters_out, double *rel_out, cudaStream_t s);
// mlp_simt.cu -- fp32 FFMA MLP path (CRVPINN_PREC_FP32)
struct MlpPlan {
    long offW[CRV_MAX_LAYERS], offB[CRV_MAX_LAYERS];   // partial-buffer offsets per layer
    int splitW[CRV_MAX_LAYERS];                       // K-splits of the weight-gradient GEMM
    int cs_split;                                     // row chunks of the column reductions
    int rows_per;
    long partial_floats;
    int njobs, max_count, groups;
    RedJob jobs[2 * CRV_MAX_LAYERS];
};
struct SimtBufs {
    float *act;        // [hidden a=1..L][P][w_a] fp32, slot stride P*wmax
    float *delta0, *delta1;
    float *gbar;       // [P]
    float *partial;    // reduction partials (MlpPlan)
    const RedJob *jobs;// device copy of plan.jobs
};
void simt_make_plan(const Net &net, MlpPlan &plan);
void simt_forward(const Net &net, const float *theta, const SimtBufs &b, float *u, cudaStream_t s);
void simt_eval_points(const Net &net, const float *theta, const SimtBufs &b, const float *xy, int npts,
                      float *out, cudaStream_t s);
void simt_backward(const Net &net, const MlpPlan &plan, const float *theta, const SimtBufs &b,
                   float *grad, cudaStream_t s);
int simt_launches_fwd(const Net &net);
int simt_launches_bwd(const Net &net);
}  // namespace crv
