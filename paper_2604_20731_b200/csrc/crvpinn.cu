// crvpinn.cu -- host side of the C ABI (include/crvpinn.h): context, device buffers, the
// per-iteration launch sequence (A1..A8) and its CUDA-graph capture.
#include "../../include/crvpinn.h"
#include "common.cuh"
#include "mlp_tc.cuh"

#include <dlfcn.h>
#include <nccl.h>   // types only: libnccl.so.2 is opened on first use (sharded contexts)

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

using namespace crv;

namespace {

std::string g_err;   // errors raised before a context exists

// NCCL entry points, resolved from libnccl.so.2 at the first sharded create / unique-id call. The
// library itself has no link-time NCCL dependency (a process that already loaded torch's NCCL gets
// that same copy: dlopen matches the soname).
struct NcclApi {
    bool tried = false, ok = false;
    std::string err;
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char *e = dlerror();
        g_nccl.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
        return false;
    }
    g_nccl.get_unique_id = (decltype(g_nccl.get_unique_id))dlsym(h, "ncclGetUniqueId");
    g_nccl.comm_init_rank = (decltype(g_nccl.comm_init_rank))dlsym(h, "ncclCommInitRank");
    g_nccl.all_reduce = (decltype(g_nccl.all_reduce))dlsym(h, "ncclAllReduce");
    g_nccl.comm_destroy = (decltype(g_nccl.comm_destroy))dlsym(h, "ncclCommDestroy");
    g_nccl.error_string = (decltype(g_nccl.error_string))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.all_reduce && g_nccl.comm_destroy &&
                g_nccl.error_string;
    if (!g_nccl.ok) g_nccl.err = "libnccl.so.2 lacks ncclGetUniqueId/ncclCommInitRank/ncclAllReduce";
    return g_nccl.ok;
}

// balanced split of T tiles over w shards (crvpinn_shard_tiles)
void shard_split(long T, int r, int w, long &t0, long &nt) {
    t0 = (long)((long long)r * T / w);
    nt = (long)((long long)(r + 1) * T / w) - t0;
}

struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    double *hist = nullptr;               // device loss history of this graph's n iterations
    std::vector<cudaEvent_t> ev;          // 5 per iteration when captured with profiling
};

}  // namespace

struct crvpinn_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    crvpinn_opts opts{};
    Net net{};
    long np = 0;
    // fields
    float *K = nullptr, *S = nullptr, *f = nullptr, *alpha = nullptr, *b = nullptr;
    float *u = nullptr, *res = nullptr, *q = nullptr, *gu_lat = nullptr;
    GramConsts gram{};
    double *loss_part = nullptr;
    int loss_nblk = 0;
    DevState *st = nullptr, *snap_st = nullptr;
    float *theta = nullptr, *m = nullptr, *v = nullptr, *grad = nullptr;
    float *snap_theta = nullptr, *snap_m = nullptr, *snap_v = nullptr;
    // MLP buffers
    SimtBufs simt{};
    MlpPlan plan{};
    RedJob *d_jobs = nullptr;
    TcBufs tc{};
    // host staging (pinned)
    float *h_field = nullptr;
    double *h_hist = nullptr;
    int h_hist_cap = 0;
    DevState *h_state = nullptr;
    // graphs and profiling
    std::map<int, GraphEntry> graphs;
    bool profiling = false;
    double prof_ms[4] = {0, 0, 0, 0};
    int64_t prof_iters = 0;
    std::string err;
    std::vector<void *> allocs;
    // crvpinn_eval_points: two chunks in flight, each with device xy + p, pinned host xy + p, and
    // events; a copy stream moves chunk c+1 in and chunk c-1 out while chunk c computes
    float *pts = nullptr;                 // device [2][3 * EP_CHUNK]
    float *pts_h = nullptr;               // pinned [2][3 * EP_CHUNK]
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ep_in[2] = {}, ep_done[2] = {}, ep_out[2] = {};
    float *ds_u = nullptr;         // crvpinn_direct_solve's lattice result (first use)
    // point sharding (f4): this context's tiles, and the communicator of the two exchanges
    long tile0 = 0, ntiles = 0;
    bool sharded = false;          // shard_world > 1 or a communicator: u is zeroed before the forward
    ncclComm_t comm = nullptr;
    ncclResult_t nccl_rc = ncclSuccess;   // first failed NCCL call of a launch sequence
};

#define CK(call)                                                                 \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);      \
            return CRVPINN_ECUDA;                                                \
        }                                                                        \
    } while (0)

static int fail(crvpinn_ctx *ctx, int code, const std::string &msg) {
    if (ctx) ctx->err = msg; else g_err = msg;
    return code;
}

template <class T>
static int dalloc(crvpinn_ctx *ctx, T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T) > 0 ? count * sizeof(T) : 16);
    if (e != cudaSuccess) {
        ctx->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
        return e == cudaErrorMemoryAllocation ? CRVPINN_ENOMEM : CRVPINN_ECUDA;
    }
    // zero-filled on the context stream: a cudaMemset on the legacy stream is not ordered with the
    // (non-blocking) context stream and could land after a later copy or kernel there wrote the buffer
    cudaMemsetAsync(q, 0, count * sizeof(T) > 0 ? count * sizeof(T) : 16, ctx->stream);
    ctx->allocs.push_back(q);
    *p = (T *)q;
    return CRVPINN_OK;
}

#define DALLOC(ptr, count)                                   \
    do {                                                     \
        int rc_ = dalloc(ctx, &(ptr), (size_t)(count));      \
        if (rc_ != CRVPINN_OK) return rc_;                   \
    } while (0)

// ---------------------------------------------------------------- one iteration
// Launches A1..A8 on the context stream. train = 0: evaluation only (no Adam, t unchanged).
// Event-record nodes inside a captured graph need cudaEventRecordExternal (a plain record during
// capture only expresses a dependency and is never executed as a timestamp).
static void record(cudaEvent_t e, cudaStream_t s) { cudaEventRecordWithFlags(e, s, cudaEventRecordExternal); }

// sum over the shards, in place, on the context stream (a no-op without a communicator)
static void exchange(crvpinn_ctx *ctx, float *buf, size_t count) {
    if (!ctx->comm) return;
    ncclResult_t r = g_nccl.all_reduce(buf, buf, count, ncclFloat32, ncclSum, ctx->comm, ctx->stream);
    if (r != ncclSuccess && ctx->nccl_rc == ncclSuccess) ctx->nccl_rc = r;
}

static size_t lattice_count(const crvpinn_ctx *ctx) { return (size_t)(ctx->net.N + 1) * (ctx->net.N + 1); }

// A1 on this context's points (all of them unsharded); sharded: into a zeroed field
static void launch_forward(crvpinn_ctx *ctx) {
    cudaStream_t s = ctx->stream;
    if (ctx->sharded) cudaMemsetAsync(ctx->u, 0, sizeof(float) * lattice_count(ctx), s);
    if (ctx->opts.precision == CRVPINN_PREC_TENSOR) tc_forward(ctx->net, ctx->tc, ctx->u, s);
    else simt_forward(ctx->net, ctx->theta, ctx->simt, ctx->u, s);
}

// A8 on the tensor path after the gradient all-reduce (sharded contexts with a communicator)
static void tc_adam_after_exchange(crvpinn_ctx *ctx) {
    const AdamOp A = tc_adam_op(ctx->net, ctx->tc, ctx->theta, ctx->m, ctx->v, ctx->st, (float)ctx->opts.lr,
                                (float)ctx->opts.beta1, (float)ctx->opts.beta2, (float)ctx->opts.eps);
    launch_adam_op(ctx->grad, ctx->np, A, ctx->stream);
}

// fwd = false: u is already in place (crvpinn_shard_backward); xchg: the two all-reduces
static void launch_iteration(crvpinn_ctx *ctx, double *hist, int n_hist, bool train, cudaEvent_t *ev,
                             bool fwd = true, bool xchg = true) {
    cudaStream_t s = ctx->stream;
    const Net &net = ctx->net;
    const bool tc = ctx->opts.precision == CRVPINN_PREC_TENSOR;
    if (ev) record(ev[0], s);
    // A1: network at every MLP point of this shard -> u on the lattice; sharded: sum over shards
    if (fwd) launch_forward(ctx);
    if (fwd && xchg) exchange(ctx, ctx->u, lattice_count(ctx));
    if (ev) record(ev[1], s);
    // A2-A5: residual, Gram solve, loss, adjoint
    float *gbar = tc ? ctx->tc.gbar : ctx->simt.gbar;
    launch_field_chain(ctx->u, ctx->alpha, ctx->b, ctx->res, ctx->q, gbar, ctx->gu_lat, ctx->loss_part, ctx->gram,
                       net.N, ctx->st, tc ? 1 : 0, hist, n_hist, ctx->opts.beta1, ctx->opts.beta2, train ? 1 : 0, s);
    if (ev) record(ev[2], s);
    // A6-A7: backward and deterministic weight-gradient reduction; tensor path: A8 (Adam + the operand
    // copies) fused into the reductions, unless the gradient is exchanged first (sharded)
    const bool fuse_adam = tc && train && !ctx->comm;
    if (tc) {
        AdamOp A{};
        if (fuse_adam)
            A = tc_adam_op(net, ctx->tc, ctx->theta, ctx->m, ctx->v, ctx->st, (float)ctx->opts.lr,
                           (float)ctx->opts.beta1, (float)ctx->opts.beta2, (float)ctx->opts.eps);
        tc_backward(net, ctx->tc, ctx->st, ctx->grad, s, &A);
    } else {
        simt_backward(net, ctx->plan, ctx->theta, ctx->simt, ctx->grad, s);
    }
    if (xchg) exchange(ctx, ctx->grad, (size_t)ctx->np);   // each shard holds its points' share
    if (ev) record(ev[3], s);
    // A8: Adam (fp32 path; tensor path with a communicator: after the gradient exchange)
    if (train && !fuse_adam) {
        if (tc)
            tc_adam_after_exchange(ctx);
        else
            launch_adam(ctx->theta, ctx->m, ctx->v, ctx->grad, ctx->np, ctx->st, ctx->st,
                        (float)ctx->opts.lr, (float)ctx->opts.beta1, (float)ctx->opts.beta2,
                        (float)ctx->opts.eps, s);
    }
    if (ev) record(ev[4], s);
}

static int launches_per_iter(const crvpinn_ctx *ctx) {
    const bool tc = ctx->opts.precision == CRVPINN_PREC_TENSOR;
    int mlp = tc ? tc_launches(ctx->net, ctx->tc) : simt_launches_fwd(ctx->net) + simt_launches_bwd(ctx->net);
    // (sharded: + the memset of u and the two NCCL all-reduce kernels, which are not ours)
    const bool fused = tc && !ctx->comm;   // tensor path: Adam inside the reductions
    return mlp + 4 /*residual+DST, tridiagonal, inverse DST+loss, adjoint+loss final*/ + (fused ? 0 : 1) /*adam*/;
}

static void drop_graphs(crvpinn_ctx *ctx) {
    for (auto &kv : ctx->graphs) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.hist) cudaFree(kv.second.hist);
        for (auto e : kv.second.ev) cudaEventDestroy(e);
    }
    ctx->graphs.clear();
}

static int snapshot_copies(crvpinn_ctx *ctx, bool to_snap) {
    cudaStream_t s = ctx->stream;
    size_t bytes = sizeof(float) * ctx->np;
    float *a[3] = {ctx->theta, ctx->m, ctx->v}, *b[3] = {ctx->snap_theta, ctx->snap_m, ctx->snap_v};
    for (int k = 0; k < 3; ++k)
        CK(cudaMemcpyAsync(to_snap ? b[k] : a[k], to_snap ? a[k] : b[k], bytes, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(to_snap ? ctx->snap_st : ctx->st, to_snap ? ctx->st : ctx->snap_st, sizeof(DevState),
                       cudaMemcpyDeviceToDevice, s));
    return CRVPINN_OK;
}

static int get_graph(crvpinn_ctx *ctx, int n, GraphEntry **out) {
    auto it = ctx->graphs.find(n);
    if (it != ctx->graphs.end()) { *out = &it->second; return CRVPINN_OK; }
    GraphEntry ge;
    CK(cudaMalloc(&ge.hist, sizeof(double) * (size_t)n));
    if (ctx->profiling) {
        ge.ev.resize((size_t)5 * n);
        for (auto &e : ge.ev) CK(cudaEventCreate(&e));
    }
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    launch_begin_call(ctx->st, ctx->stream);
    int rc = snapshot_copies(ctx, true);
    // the fp16 weight copies' exponents for this call: room for n Adam steps
    if (ctx->opts.precision == CRVPINN_PREC_TENSOR)
        tc_refresh_weights(ctx->net, ctx->tc, ctx->theta, ctx->st, (float)(4.0 * n * ctx->opts.lr), ctx->stream);
    for (int k = 0; k < n && rc == CRVPINN_OK; ++k)
        launch_iteration(ctx, ge.hist, n, true, ctx->profiling ? &ge.ev[(size_t)5 * k] : nullptr);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
    if (rc != CRVPINN_OK) return rc;
    if (ctx->nccl_rc != ncclSuccess) {
        if (g) cudaGraphDestroy(g);
        return fail(ctx, CRVPINN_ECUDA, std::string("NCCL all-reduce in graph capture: ") +
                                            g_nccl.error_string(ctx->nccl_rc));
    }
    if (e != cudaSuccess) return fail(ctx, CRVPINN_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&ge.exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(ctx, CRVPINN_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    ctx->graphs[n] = ge;
    *out = &ctx->graphs[n];
    return CRVPINN_OK;
}

static bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

static uint64_t splitmix(uint64_t &s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static int check_field(crvpinn_ctx *ctx, const float *F, int N, bool positive, const char *name) {
    long nn = (long)(N + 1) * (N + 1);
    for (long i = 0; i < nn; ++i) {
        float x = F[i];
        if (!std::isfinite(x) || (positive && !(x > 0.0f)))
            return fail(ctx, CRVPINN_EDOMAIN, std::string(name) + (positive ? " must be finite and > 0" : " must be finite"));
    }
    return CRVPINN_OK;
}

static int upload_field(crvpinn_ctx *ctx, float *dst, const float *src) {
    size_t bytes = sizeof(float) * (size_t)(ctx->net.N + 1) * (ctx->net.N + 1);
    CK(cudaStreamSynchronize(ctx->stream));   // staging buffer reuse
    memcpy(ctx->h_field, src, bytes);
    CK(cudaMemcpyAsync(dst, ctx->h_field, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return CRVPINN_OK;
}

extern "C" {

void crvpinn_default_opts(crvpinn_opts *o) {
    if (!o) return;
    o->lr = 1e-3;
    o->beta1 = 0.9;
    o->beta2 = 0.999;
    o->eps = 1e-8;
    o->mobility_ratio = 25.35 / 3.95;
    o->precision = CRVPINN_PREC_TENSOR;
    o->seed = 0;
    o->stream = nullptr;
    o->device = 0;
    o->gravity = 0.0;
    o->density_ratio = 479.0 / 1045.0;
    o->shard_rank = 0;
    o->shard_world = 1;
    o->nccl = 0;
    memset(o->nccl_id, 0, sizeof(o->nccl_id));
}

const char *crvpinn_last_error(const crvpinn_ctx *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

size_t crvpinn_num_params(const crvpinn_ctx *ctx) { return ctx ? (size_t)ctx->np : 0; }

void *crvpinn_stream(const crvpinn_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int crvpinn_launches_per_iter(const crvpinn_ctx *ctx) { return ctx ? launches_per_iter(ctx) : 0; }

void crvpinn_destroy(crvpinn_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    drop_graphs(ctx);
    if (ctx->comm) g_nccl.comm_destroy(ctx->comm);
    gram_free_constants(ctx->gram);
    tc_destroy(ctx->tc);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
    if (ctx->pts) cudaFree(ctx->pts);
    if (ctx->pts_h) cudaFreeHost(ctx->pts_h);
    for (int b = 0; b < 2; ++b) {
        if (ctx->ep_in[b]) cudaEventDestroy(ctx->ep_in[b]);
        if (ctx->ep_done[b]) cudaEventDestroy(ctx->ep_done[b]);
        if (ctx->ep_out[b]) cudaEventDestroy(ctx->ep_out[b]);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (void *p : ctx->allocs) cudaFree(p);
    if (ctx->h_field) cudaFreeHost(ctx->h_field);
    if (ctx->h_hist) cudaFreeHost(ctx->h_hist);
    if (ctx->h_state) cudaFreeHost(ctx->h_state);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

static int create_impl(crvpinn_ctx *ctx, int N, int n_widths, const int *widths, const float *K,
                       const float *S, const float *f, const float *theta0) {
    // ---- geometry
    Net &net = ctx->net;
    net.N = N; net.n = N - 1; net.P = N * N; net.nl = n_widths - 1;
    long np = 0;
    for (int l = 0; l < n_widths; ++l) net.widths[l] = widths[l];
    for (int l = 0; l < net.nl; ++l) {
        net.woff[l] = np; np += (long)widths[l + 1] * widths[l];
        net.boff[l] = np; np += widths[l + 1];
    }
    ctx->np = np;
    // ---- device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= ctx->opts.device)
        return fail(ctx, CRVPINN_ECUDA, "no CUDA device available (this library has no CPU fallback)");
    CK(cudaSetDevice(ctx->opts.device));
    ctx->device = ctx->opts.device;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, ctx->device));
    if (prop.major != 10)
        return fail(ctx, CRVPINN_ECUDA, "device is not sm_100 (B200); this build targets sm_100a only");
    if (ctx->opts.stream) {
        ctx->stream = (cudaStream_t)ctx->opts.stream;
    } else {
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    long nn = (long)(N + 1) * (N + 1);
    int n = N - 1;
    DALLOC(ctx->K, nn); DALLOC(ctx->S, nn); DALLOC(ctx->f, nn);
    DALLOC(ctx->alpha, nn); DALLOC(ctx->b, nn); DALLOC(ctx->u, nn); DALLOC(ctx->gu_lat, nn);
    DALLOC(ctx->res, (long)n * n); DALLOC(ctx->q, (long)n * n);
    ctx->gram = gram_make_constants(N);
    if (!ctx->gram.etab || !ctx->gram.work) return fail(ctx, CRVPINN_ENOMEM, "Gram constants allocation failed");
    ctx->loss_nblk = field_chain_loss_blocks(N);
    DALLOC(ctx->loss_part, ctx->loss_nblk);
    DALLOC(ctx->st, 1); DALLOC(ctx->snap_st, 1);
    DALLOC(ctx->theta, np); DALLOC(ctx->m, np); DALLOC(ctx->v, np); DALLOC(ctx->grad, np);
    DALLOC(ctx->snap_theta, np); DALLOC(ctx->snap_m, np); DALLOC(ctx->snap_v, np);
    CK(cudaMallocHost(&ctx->h_field, sizeof(float) * nn));
    CK(cudaMallocHost(&ctx->h_state, sizeof(DevState)));
    // ---- MLP buffers
    int wmax = 0;
    for (int l = 1; l < net.nl; ++l) wmax = widths[l] > wmax ? widths[l] : wmax;
    if (ctx->opts.precision == CRVPINN_PREC_FP32) {
        simt_make_plan(net, ctx->plan);
        DALLOC(ctx->simt.act, (long)(net.nl - 1) * net.P * wmax);
        DALLOC(ctx->simt.delta0, (long)net.P * wmax);
        DALLOC(ctx->simt.delta1, (long)net.P * wmax);
        DALLOC(ctx->simt.gbar, net.P);
        DALLOC(ctx->simt.partial, ctx->plan.partial_floats);
        DALLOC(ctx->d_jobs, ctx->plan.njobs);
        CK(cudaMemcpyAsync(ctx->d_jobs, ctx->plan.jobs, sizeof(RedJob) * ctx->plan.njobs, cudaMemcpyHostToDevice,
                           ctx->stream));
        ctx->simt.jobs = ctx->d_jobs;
    } else {
        int rc = tc_create(net, ctx->tc, (int)ctx->tile0, (int)ctx->ntiles, ctx->err);
        if (rc != 0) return rc;
        ctx->tc.st = ctx->st;
    }
    // ---- inputs, A0, Gram constants
    std::vector<float> th((size_t)np);
    if (theta0) {
        memcpy(th.data(), theta0, sizeof(float) * np);
    } else {
        uint64_t sd = ctx->opts.seed;
        for (int l = 0; l < net.nl; ++l) {
            int fin = widths[l], fout = widths[l + 1];
            double a = std::sqrt(6.0 / (fin + fout));
            for (long k = 0; k < (long)fin * fout; ++k) {
                double r = (double)(splitmix(sd) >> 11) * (1.0 / 9007199254740992.0);
                th[net.woff[l] + k] = (float)((2.0 * r - 1.0) * a);
            }
            for (int k = 0; k < fout; ++k) th[net.boff[l] + k] = 0.0f;
        }
    }
    // the legacy-stream work of the set-up above (tc_create's and the Gram constants' zero fills and
    // table copies) is complete before anything on the context stream touches those buffers
    CK(cudaDeviceSynchronize());
    // pageable sources: the copies are staged and ordered on the context stream, ahead of the
    // kernels that read them (a plain cudaMemcpy runs on the legacy stream, which a non-blocking
    // context stream does not wait for)
    CK(cudaMemcpyAsync(ctx->theta, th.data(), sizeof(float) * np, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->K, K, sizeof(float) * nn, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->S, S, sizeof(float) * nn, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->f, f, sizeof(float) * nn, cudaMemcpyHostToDevice, ctx->stream));
    launch_alpha(ctx->K, ctx->S, ctx->alpha, N, (float)ctx->opts.mobility_ratio, ctx->stream);
    launch_rhs(ctx->K, ctx->S, ctx->f, ctx->b, N, (float)ctx->opts.mobility_ratio, (float)ctx->opts.density_ratio,
               (float)ctx->opts.gravity, ctx->stream);
    if (ctx->opts.precision == CRVPINN_PREC_TENSOR) tc_refresh_weights(net, ctx->tc, ctx->theta, ctx->st, 0.0f, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    // ---- the shards' communicator (collective: every rank creates its context concurrently)
    if (ctx->opts.nccl) {
        ncclUniqueId id;
        memcpy(&id, ctx->opts.nccl_id, sizeof(id) < 128 ? sizeof(id) : 128);
        ncclResult_t r = g_nccl.comm_init_rank(&ctx->comm, ctx->opts.shard_world, id, ctx->opts.shard_rank);
        if (r != ncclSuccess) {
            ctx->comm = nullptr;
            return fail(ctx, CRVPINN_ECUDA, std::string("ncclCommInitRank: ") + g_nccl.error_string(r));
        }
    }
    return CRVPINN_OK;
}

int crvpinn_create(crvpinn_ctx **out, int N, int n_widths, const int *widths, const float *K,
                   const float *S, const float *f, const float *theta0, const crvpinn_opts *opts) {
    if (!out) return fail(nullptr, CRVPINN_EINVAL, "out is NULL");
    *out = nullptr;
    if (!widths || !K || !S || !f) return fail(nullptr, CRVPINN_EINVAL, "widths, K, S, f are required");
    if (!is_pow2(N) || N < 16 || N > 2048) return fail(nullptr, CRVPINN_EINVAL, "N must be a power of two in [16, 2048]");
    if (n_widths < 3 || n_widths > CRV_MAX_LAYERS + 1) return fail(nullptr, CRVPINN_EINVAL, "need 3..17 widths");
    if (widths[0] != 2 || widths[n_widths - 1] != 1) return fail(nullptr, CRVPINN_EINVAL, "widths must be {2, ..., 1}");
    for (int l = 1; l < n_widths - 1; ++l)
        if (widths[l] < 32 || widths[l] > 256 || widths[l] % 32 != 0)
            return fail(nullptr, CRVPINN_EINVAL, "hidden widths must be multiples of 32 in [32, 256]");
    crvpinn_ctx *ctx = new crvpinn_ctx();
    if (opts) ctx->opts = *opts; else crvpinn_default_opts(&ctx->opts);
    {
        const int w = ctx->opts.shard_world, r = ctx->opts.shard_rank;
        const long T = (long)N * N / 128;
        if (w < 1 || r < 0 || r >= w || w > T) {
            delete ctx;
            return fail(nullptr, CRVPINN_EINVAL, "need 0 <= shard_rank < shard_world <= N*N/128");
        }
        if (w > 1 && ctx->opts.precision != CRVPINN_PREC_TENSOR) {
            delete ctx;
            return fail(nullptr, CRVPINN_EINVAL, "point sharding needs the tensor path");
        }
        if (ctx->opts.nccl && !nccl_load()) {
            delete ctx;
            return fail(nullptr, CRVPINN_ECUDA, g_nccl.err);
        }
        shard_split(T, r, w, ctx->tile0, ctx->ntiles);
        ctx->sharded = w > 1 || ctx->opts.nccl;
    }
    if (!std::isfinite(ctx->opts.gravity) || !std::isfinite(ctx->opts.density_ratio) || ctx->opts.density_ratio < 0.0) {
        delete ctx;
        return fail(nullptr, CRVPINN_EINVAL, "gravity / density_ratio must be finite (density_ratio >= 0)");
    }
    if (ctx->opts.precision == CRVPINN_PREC_TENSOR) {
        for (int l = 2; l < n_widths - 1; ++l)
            if (widths[l] != widths[1]) {
                delete ctx;
                return fail(nullptr, CRVPINN_EINVAL, "tensor path needs equal hidden widths");
            }
    } else if (ctx->opts.precision != CRVPINN_PREC_FP32) {
        delete ctx;
        return fail(nullptr, CRVPINN_EINVAL, "unknown precision");
    }
    int rc = check_field(ctx, K, N, true, "K");
    if (rc == CRVPINN_OK) rc = check_field(ctx, S, N, false, "S");
    if (rc == CRVPINN_OK) rc = check_field(ctx, f, N, false, "f");
    if (rc == CRVPINN_OK) rc = create_impl(ctx, N, n_widths, widths, K, S, f, theta0);
    if (rc != CRVPINN_OK) {
        g_err = ctx->err;
        crvpinn_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return CRVPINN_OK;
}

int crvpinn_set_saturation(crvpinn_ctx *ctx, const float *S) {
    if (!ctx || !S) return fail(ctx, CRVPINN_EINVAL, "null argument");
    int rc = check_field(ctx, S, ctx->net.N, false, "S");
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    rc = upload_field(ctx, ctx->S, S);
    if (rc) return rc;
    launch_alpha(ctx->K, ctx->S, ctx->alpha, ctx->net.N, (float)ctx->opts.mobility_ratio, ctx->stream);
    launch_rhs(ctx->K, ctx->S, ctx->f, ctx->b, ctx->net.N, (float)ctx->opts.mobility_ratio,
               (float)ctx->opts.density_ratio, (float)ctx->opts.gravity, ctx->stream);
    CK(cudaGetLastError());
    return CRVPINN_OK;
}

int crvpinn_set_saturation_device(crvpinn_ctx *ctx, const void *S_dev) {
    if (!ctx || !S_dev) return fail(ctx, CRVPINN_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device));
    size_t bytes = sizeof(float) * (size_t)(ctx->net.N + 1) * (ctx->net.N + 1);
    CK(cudaMemcpyAsync(ctx->S, S_dev, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    launch_alpha(ctx->K, ctx->S, ctx->alpha, ctx->net.N, (float)ctx->opts.mobility_ratio, ctx->stream);
    launch_rhs(ctx->K, ctx->S, ctx->f, ctx->b, ctx->net.N, (float)ctx->opts.mobility_ratio,
               (float)ctx->opts.density_ratio, (float)ctx->opts.gravity, ctx->stream);
    CK(cudaGetLastError());
    return CRVPINN_OK;
}

static bool needs_caller_exchange(const crvpinn_ctx *ctx) { return ctx->opts.shard_world > 1 && !ctx->comm; }

int crvpinn_step(crvpinn_ctx *ctx, int n_adam, double *loss_hist) {
    if (!ctx || n_adam < 1) return fail(ctx, CRVPINN_EINVAL, "n_adam must be >= 1");
    if (needs_caller_exchange(ctx))
        return fail(ctx, CRVPINN_EINVAL, "sharded context without a communicator: use crvpinn_shard_forward/backward");
    CK(cudaSetDevice(ctx->device));
    GraphEntry *ge = nullptr;
    int rc = get_graph(ctx, n_adam, &ge);
    if (rc) return rc;
    CK(cudaGraphLaunch(ge->exec, ctx->stream));
    if (loss_hist) {
        if (ctx->h_hist_cap < n_adam) {
            if (ctx->h_hist) cudaFreeHost(ctx->h_hist);
            CK(cudaMallocHost(&ctx->h_hist, sizeof(double) * n_adam));
            ctx->h_hist_cap = n_adam;
        }
        CK(cudaMemcpyAsync(ctx->h_hist, ge->hist, sizeof(double) * n_adam, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaMemcpyAsync(ctx->h_state, ctx->st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    if (loss_hist) memcpy(loss_hist, ctx->h_hist, sizeof(double) * n_adam);
    if (ctx->profiling) {
        for (int k = 0; k < n_adam; ++k)
            for (int s = 0; s < 4; ++s) {
                float ms = 0.0f;
                CK(cudaEventElapsedTime(&ms, ge->ev[(size_t)5 * k + s], ge->ev[(size_t)5 * k + s + 1]));
                ctx->prof_ms[s] += ms;
            }
        ctx->prof_iters += n_adam;
    }
    if (ctx->h_state->nonfinite) {
        rc = snapshot_copies(ctx, false);
        if (rc) return rc;
        // the tensor path computes only from its fp16 weight copies, which every Adam step of the
        // call rewrote: rebuild them from the restored theta
        if (ctx->opts.precision == CRVPINN_PREC_TENSOR) tc_refresh_weights(ctx->net, ctx->tc, ctx->theta, ctx->st, 0.0f, ctx->stream);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(ctx->stream));
        return fail(ctx, CRVPINN_ENONFINITE, "non-finite loss or gradient; theta and Adam state restored");
    }
    return CRVPINN_OK;
}

int crvpinn_pretrain(crvpinn_ctx *ctx, int n_iters, double *loss_hist) {
    return crvpinn_step(ctx, n_iters, loss_hist);
}

int crvpinn_eval(crvpinn_ctx *ctx, float *p_out) {
    if (!ctx || !p_out) return fail(ctx, CRVPINN_EINVAL, "null argument");
    if (needs_caller_exchange(ctx))
        return fail(ctx, CRVPINN_EINVAL, "sharded context without a communicator: use crvpinn_shard_forward");
    CK(cudaSetDevice(ctx->device));
    ctx->nccl_rc = ncclSuccess;
    launch_forward(ctx);
    exchange(ctx, ctx->u, lattice_count(ctx));
    if (ctx->nccl_rc != ncclSuccess)
        return fail(ctx, CRVPINN_ECUDA, std::string("NCCL all-reduce: ") + g_nccl.error_string(ctx->nccl_rc));
    size_t nn = (size_t)(ctx->net.N + 1) * (ctx->net.N + 1);
    CK(cudaMemcpyAsync(ctx->h_field, ctx->u, sizeof(float) * nn, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    memcpy(p_out, ctx->h_field, sizeof(float) * nn);
    return CRVPINN_OK;
}

constexpr long EP_CHUNK = 1L << 18;   // points per chunk (a multiple of the 128-point tile)

int crvpinn_eval_points(crvpinn_ctx *ctx, long n, const float *xy, float *p_out) {
    if (!ctx) return fail(ctx, CRVPINN_EINVAL, "null ctx");
    if (n < 0) return fail(ctx, CRVPINN_EINVAL, "n must be >= 0");
    if (n == 0) return CRVPINN_OK;
    if (!xy || !p_out) return fail(ctx, CRVPINN_EINVAL, "null argument");
    if (n > (1L << 30)) return fail(ctx, CRVPINN_EINVAL, "too many points in one call (max 2^30)");
    {   // branch-free scan (vectorises): a float is non-finite iff its exponent bits are all set
        const uint32_t *w = reinterpret_cast<const uint32_t *>(xy);
        uint32_t bad = 0;
        for (long i = 0; i < 2 * n; ++i) bad |= (uint32_t)((w[i] & 0x7f800000u) == 0x7f800000u);
        if (bad) return fail(ctx, CRVPINN_EDOMAIN, "non-finite coordinate");
    }
    CK(cudaSetDevice(ctx->device));
    if (!ctx->pts) {
        CK(cudaMalloc(&ctx->pts, sizeof(float) * 6 * (size_t)EP_CHUNK));
        CK(cudaMallocHost(&ctx->pts_h, sizeof(float) * 6 * (size_t)EP_CHUNK));
        CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CK(cudaEventCreateWithFlags(&ctx->ep_in[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ep_done[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ep_out[b], cudaEventDisableTiming));
        }
    }
    CK(cudaStreamSynchronize(ctx->stream));   // the weights of any queued training are final
    const long nch = (n + EP_CHUNK - 1) / EP_CHUNK;
    auto drain = [&](long c) -> int {          // chunk c's values -> p_out (host)
        const int b = (int)(c & 1);
        const long c0 = c * EP_CHUNK, cn = n - c0 < EP_CHUNK ? n - c0 : EP_CHUNK;
        CK(cudaEventSynchronize(ctx->ep_out[b]));
        memcpy(p_out + c0, ctx->pts_h + (size_t)b * 3 * EP_CHUNK + 2 * EP_CHUNK, sizeof(float) * cn);
        return CRVPINN_OK;
    };
    for (long c = 0; c < nch; ++c) {
        const int b = (int)(c & 1);
        const long c0 = c * EP_CHUNK, cn = n - c0 < EP_CHUNK ? n - c0 : EP_CHUNK;
        float *hb = ctx->pts_h + (size_t)b * 3 * EP_CHUNK, *db = ctx->pts + (size_t)b * 3 * EP_CHUNK;
        if (c >= 2) {   // buffer b last held chunk c-2: its result must be out before it is reused
            int rc = drain(c - 2);
            if (rc) return rc;
        }
        memcpy(hb, xy + 2 * c0, sizeof(float) * 2 * cn);   // pageable -> pinned, overlapping the GPU
        CK(cudaMemcpyAsync(db, hb, sizeof(float) * 2 * cn, cudaMemcpyHostToDevice, ctx->copy_stream));
        CK(cudaEventRecord(ctx->ep_in[b], ctx->copy_stream));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ep_in[b], 0));
        if (ctx->opts.precision == CRVPINN_PREC_TENSOR)
            tc_eval_points(ctx->net, ctx->tc, db, (int)cn, db + 2 * EP_CHUNK, ctx->stream);
        else
            simt_eval_points(ctx->net, ctx->theta, ctx->simt, db, (int)cn, db + 2 * EP_CHUNK, ctx->stream);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ctx->ep_done[b], ctx->stream));
        CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ep_done[b], 0));
        CK(cudaMemcpyAsync(hb + 2 * EP_CHUNK, db + 2 * EP_CHUNK, sizeof(float) * cn, cudaMemcpyDeviceToHost,
                           ctx->copy_stream));
        CK(cudaEventRecord(ctx->ep_out[b], ctx->copy_stream));
    }
    for (long c = nch >= 2 ? nch - 2 : 0; c < nch; ++c) {
        int rc = drain(c);
        if (rc) return rc;
    }
    CK(cudaStreamSynchronize(ctx->copy_stream));
    return CRVPINN_OK;
}

int crvpinn_direct_solve(crvpinn_ctx *ctx, double rtol, int max_iter, float *u_out, int *iters, double *rel_res) {
    if (!ctx) return fail(ctx, CRVPINN_EINVAL, "null ctx");
    if (!(rtol > 0.0) || max_iter < 1) return fail(ctx, CRVPINN_EINVAL, "need rtol > 0 and max_iter >= 1");
    CK(cudaSetDevice(ctx->device));
    const int N = ctx->net.N;
    const size_t nn = (size_t)(N + 1) * (N + 1);
    if (!ctx->ds_u) DALLOC(ctx->ds_u, nn);   // lattice result (boundary 0), apart from the training buffers
    float *ud = ctx->ds_u;
    CK(cudaMemsetAsync(ud, 0, sizeof(float) * nn, ctx->stream));
    int it = 0;
    double rel = 0.0;
    const int prc = pcg_solve(ctx->alpha, ctx->b, ud, ctx->gram, N, rtol, max_iter, &it, &rel, ctx->stream);
    cudaError_t e = cudaSuccess;
    if (prc == 0 && u_out) {
        e = cudaMemcpyAsync(ctx->h_field, ud, sizeof(float) * nn, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e == cudaSuccess) memcpy(u_out, ctx->h_field, sizeof(float) * nn);
    }
    if (prc != 0 || e != cudaSuccess) {
        ctx->err = std::string("direct solve: ") + cudaGetErrorString(e != cudaSuccess ? e : cudaGetLastError());
        return CRVPINN_ECUDA;
    }
    if (iters) *iters = it;
    if (rel_res) *rel_res = rel;
    if (!std::isfinite(rel)) return fail(ctx, CRVPINN_ENONFINITE, "non-finite residual in the direct solve");
    return CRVPINN_OK;
}

int crvpinn_loss_grad(crvpinn_ctx *ctx, double *loss, float *grad) {
    if (!ctx || !loss) return fail(ctx, CRVPINN_EINVAL, "null argument");
    if (needs_caller_exchange(ctx))
        return fail(ctx, CRVPINN_EINVAL, "sharded context without a communicator: use crvpinn_shard_forward/backward");
    CK(cudaSetDevice(ctx->device));
    ctx->nccl_rc = ncclSuccess;
    launch_begin_call(ctx->st, ctx->stream);
    launch_iteration(ctx, nullptr, 0, false, nullptr);
    if (ctx->nccl_rc != ncclSuccess)
        return fail(ctx, CRVPINN_ECUDA, std::string("NCCL all-reduce: ") + g_nccl.error_string(ctx->nccl_rc));
    CK(cudaMemcpyAsync(ctx->h_state, ctx->st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
    if (grad) CK(cudaMemcpyAsync(grad, ctx->grad, sizeof(float) * ctx->np, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    *loss = ctx->h_state->loss;
    if (!std::isfinite(*loss)) return fail(ctx, CRVPINN_ENONFINITE, "non-finite loss");
    return CRVPINN_OK;
}

int crvpinn_get_intermediates(crvpinn_ctx *ctx, float *u, float *res, float *q, float *gu) {
    if (!ctx) return fail(ctx, CRVPINN_EINVAL, "null ctx");
    CK(cudaSetDevice(ctx->device));
    size_t nn = (size_t)(ctx->net.N + 1) * (ctx->net.N + 1), n2 = (size_t)ctx->net.n * ctx->net.n;
    if (u) CK(cudaMemcpyAsync(u, ctx->u, sizeof(float) * nn, cudaMemcpyDeviceToHost, ctx->stream));
    if (res) CK(cudaMemcpyAsync(res, ctx->res, sizeof(float) * n2, cudaMemcpyDeviceToHost, ctx->stream));
    if (q) CK(cudaMemcpyAsync(q, ctx->q, sizeof(float) * n2, cudaMemcpyDeviceToHost, ctx->stream));
    if (gu) CK(cudaMemcpyAsync(gu, ctx->gu_lat, sizeof(float) * nn, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CRVPINN_OK;
}

int crvpinn_get_params(crvpinn_ctx *ctx, float *theta) {
    if (!ctx || !theta) return fail(ctx, CRVPINN_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(theta, ctx->theta, sizeof(float) * ctx->np, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CRVPINN_OK;
}

int crvpinn_set_params(crvpinn_ctx *ctx, const float *theta) {
    if (!ctx || !theta) return fail(ctx, CRVPINN_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(ctx->theta, theta, sizeof(float) * ctx->np, cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->opts.precision == CRVPINN_PREC_TENSOR) tc_refresh_weights(ctx->net, ctx->tc, ctx->theta, ctx->st, 0.0f, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    return CRVPINN_OK;
}

int crvpinn_get_adam(crvpinn_ctx *ctx, float *m, float *v, int64_t *t) {
    if (!ctx) return fail(ctx, CRVPINN_EINVAL, "null ctx");
    CK(cudaSetDevice(ctx->device));
    if (m) CK(cudaMemcpyAsync(m, ctx->m, sizeof(float) * ctx->np, cudaMemcpyDeviceToHost, ctx->stream));
    if (v) CK(cudaMemcpyAsync(v, ctx->v, sizeof(float) * ctx->np, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_state, ctx->st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (t) *t = ctx->h_state->t;
    return CRVPINN_OK;
}

int crvpinn_set_adam(crvpinn_ctx *ctx, const float *m, const float *v, int64_t t) {
    if (!ctx || !m || !v || t < 0) return fail(ctx, CRVPINN_EINVAL, "bad argument");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(ctx->m, m, sizeof(float) * ctx->np, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->v, v, sizeof(float) * ctx->np, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_state, ctx->st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->h_state->t = t;
    CK(cudaMemcpyAsync(ctx->st, ctx->h_state, sizeof(DevState), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CRVPINN_OK;
}

int crvpinn_set_profiling(crvpinn_ctx *ctx, int on) {
    if (!ctx) return fail(ctx, CRVPINN_EINVAL, "null ctx");
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    if ((bool)on != ctx->profiling) {
        drop_graphs(ctx);
        ctx->profiling = on != 0;
    }
    return CRVPINN_OK;
}

int crvpinn_get_profile(crvpinn_ctx *ctx, double *ms_sum, int64_t *n_iters, int reset) {
    if (!ctx) return fail(ctx, CRVPINN_EINVAL, "null ctx");
    if (ms_sum) for (int s = 0; s < 4; ++s) ms_sum[s] = ctx->prof_ms[s];
    if (n_iters) *n_iters = ctx->prof_iters;
    if (reset) {
        for (int s = 0; s < 4; ++s) ctx->prof_ms[s] = 0.0;
        ctx->prof_iters = 0;
    }
    return CRVPINN_OK;
}

int crvpinn_shard_tiles(int N, int rank, int world, long *tile0, long *ntiles) {
    if (!tile0 || !ntiles) return fail(nullptr, CRVPINN_EINVAL, "null argument");
    if (!is_pow2(N) || N < 16 || N > 2048) return fail(nullptr, CRVPINN_EINVAL, "N must be a power of two in [16, 2048]");
    const long T = (long)N * N / 128;
    if (world < 1 || rank < 0 || rank >= world || world > T)
        return fail(nullptr, CRVPINN_EINVAL, "need 0 <= rank < world <= N*N/128");
    shard_split(T, rank, world, *tile0, *ntiles);
    return CRVPINN_OK;
}

int crvpinn_nccl_unique_id(unsigned char id[128]) {
    if (!id) return fail(nullptr, CRVPINN_EINVAL, "null argument");
    if (!nccl_load()) return fail(nullptr, CRVPINN_ECUDA, g_nccl.err);
    ncclUniqueId u;
    ncclResult_t r = g_nccl.get_unique_id(&u);
    if (r != ncclSuccess) return fail(nullptr, CRVPINN_ECUDA, std::string("ncclGetUniqueId: ") + g_nccl.error_string(r));
    memset(id, 0, 128);
    memcpy(id, &u, sizeof(u) < 128 ? sizeof(u) : 128);
    return CRVPINN_OK;
}

int crvpinn_shard_forward(crvpinn_ctx *ctx, float *u_part) {
    if (!ctx || !u_part) return fail(ctx, CRVPINN_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device));
    const size_t nn = lattice_count(ctx);
    if (!ctx->sharded) CK(cudaMemsetAsync(ctx->u, 0, sizeof(float) * nn, ctx->stream));
    launch_forward(ctx);
    CK(cudaMemcpyAsync(ctx->h_field, ctx->u, sizeof(float) * nn, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    memcpy(u_part, ctx->h_field, sizeof(float) * nn);
    return CRVPINN_OK;
}

int crvpinn_shard_backward(crvpinn_ctx *ctx, const float *u_full, double *loss, float *grad_part) {
    if (!ctx || !u_full || !loss) return fail(ctx, CRVPINN_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device));
    int rc = upload_field(ctx, ctx->u, u_full);
    if (rc) return rc;
    launch_begin_call(ctx->st, ctx->stream);
    launch_iteration(ctx, nullptr, 0, false, nullptr, /*fwd=*/false, /*xchg=*/false);
    CK(cudaMemcpyAsync(ctx->h_state, ctx->st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
    if (grad_part)
        CK(cudaMemcpyAsync(grad_part, ctx->grad, sizeof(float) * ctx->np, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    *loss = ctx->h_state->loss;
    if (!std::isfinite(*loss)) return fail(ctx, CRVPINN_ENONFINITE, "non-finite loss");
    return CRVPINN_OK;
}

}  // extern "C"
