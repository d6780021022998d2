// mlp_tc.cuh -- tensor-core (tcgen05/TMEM) MLP path, CRVPINN_PREC_TENSOR.
#pragma once
#include "common.cuh"
#include <cuda_fp16.h>
#include <string>

namespace crv {

// Activation / delta storage ("tile-chunk" format): for hidden layer a, tile t
// (128 MLP points) and feature chunk c (64 features), one 16 KiB block holding 128 rows x 64
// fp16 in the UMMA SWIZZLE_128B K-major layout: element (r, f) at byte
// r*128 + (((f%64)/8) ^ (r%8))*16 + (f%8)*2. The same bytes are a valid MN-major operand
// (features contiguous), which the weight-gradient GEMM uses.
struct TcBufs {
    int ready = 0;
    int fuse_outl = 1;
    int bwd_rev = 1;         // alternate the backward launches' tile-walk direction (L2 reuse)
       // WP >= 128: output-layer backward fused into the first k_tc_bwd2 launch
    int WP = 0, KC = 0, L = 0, G = 0, ntiles = 0, tile0 = 0;   // this shard's tiles [tile0, tile0 + ntiles)
    __half *Wf = nullptr;    // [G][KC] blocks of WP rows x 128 B: B operand of the forward GEMMs
    __half *WTf = nullptr;   // [G][KC] blocks: B operand of the backward-dX GEMMs (W^T)
    float *W1p = nullptr;    // [WP][2]   first layer x 2 log2(e) (zero padded)
    float *bp = nullptr;     // [L][WP]   hidden biases x 2 log2(e) (zero padded)
    float *Wop = nullptr;    // [WP + 1]  output weights, output bias at [WP]
    __half *act = nullptr;   // [L][ntiles][KC][128*64]
    __half *delta = nullptr; // [L][ntiles][KC][128*64]  (scaled by DevState::gscale)
    float *gbar = nullptr;   // [P] dLOSS/dnet (unscaled)
    float *partial = nullptr;
    long off_ob = 0, off_dx = 0, off_dw = 0, off_cb = 0;
    int grid_ob = 0, grid_dx = 0, grid_fwd = 0, grid_bwd = 0, npairs = 0;
    int fwd_ew = 16;                       // forward epilogue warps (8: two CTAs per SM)
    RedJob *jobs = nullptr;  // device copy
    int njobs = 0, max_count = 0, groups = 0;
    int njobs_deep = 0, groups_deep = 0;   // jobs [0, njobs_deep): column sums, W1, W_out (k_reduce)
    RedJob wjobs[CRV_MAX_LAYERS];          // hidden-layer weight job of GEMM g
    bool wside[CRV_MAX_LAYERS] = {};       // ... reduced on the side stream (else inside jobs[0, njobs_deep))
    int nsm = 148;
    int chain = 0, chain_S = 0;            // backward chain (k_tc_bwdc): on/off, stages per cluster
    int cb_bias = 0;                       // hidden-layer bias gradients from the 1^T Delta partials (off_cb)
    __half *ring = nullptr;                // its per-cluster Delta rings between stages
    cudaStream_t side = nullptr;           // side stream of the per-layer weight reductions
    cudaEvent_t ev_fork[CRV_MAX_LAYERS] = {}, ev_join = nullptr;
    const float *theta = nullptr;
    DevState *st = nullptr;                // the context's device state (weight / Delta exponents)
};

// tile0, ntiles: this shard's MLP tiles [tile0, tile0 + ntiles) of net.P / 128 (the whole set unsharded);
// activations and partial sums are sized for the shard, gbar for all points
int tc_create(const Net &net, TcBufs &b, int tile0, int ntiles, std::string &err);
void tc_destroy(TcBufs &b);   // device buffers, side stream, events
void tc_forward(const Net &net, const TcBufs &b, float *u, cudaStream_t s);
// the network with cutoff at arbitrary points: out[p] = cutoff(xy[2p], xy[2p+1]) net(...), device pointers
void tc_eval_points(const Net &net, const TcBufs &b, const float *xy, int npts, float *out, cudaStream_t s);
// A6-A7, and with A (A->on) A8: Adam fused into the reductions
void tc_backward(const Net &net, const TcBufs &b, DevState *st, float *grad, cudaStream_t s,
                 const AdamOp *A = nullptr);
// fp16 copies of the hidden weights with per-layer exponents chosen for the next n Adam steps
// (margin = 4 n lr; 0 when theta does not change), plus the fp32 operand copies
void tc_refresh_weights(const Net &net, const TcBufs &b, const float *theta, DevState *st, float margin,
                        cudaStream_t s);
int tc_launches(const Net &net, const TcBufs &b);
// A8 for the tensor path, as an operation of the reductions (Adam + write of the operand copies)
AdamOp tc_adam_op(const Net &net, const TcBufs &b, float *theta, float *m, float *v, DevState *st, float lr,
                  float beta1, float beta2, float eps);

}  // namespace crv
