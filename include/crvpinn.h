/*
 * crvpinn.h -- C ABI of the B200 (sm_100a) CRVPINN pressure-update library.
 *
 * The library implements the hot path of arXiv 2604.20731 §5-§6: the robust-loss training
 * of the pressure network p_theta that replaces the MUMPS pressure solve. One Adam iteration
 * is, in the paper's notation:
 *
 *   A1 PINN_ij = 16 x(1-x) y(1-y) net_theta(x_i, y_j)            PAPER.md:373 (readings R5, R6)
 *   A2 RES_kl  = (alpha grad+ PINN, grad+ delta_kl)_h - (RHS, delta_kl)_h   Eq. 25
 *   A3 q       = G^-1 RES, G = h^-2 (4 / -1 five-point)           Eq. 26-28
 *   A4 LOSS    = RES^T q                                          Eq. 27
 *   A5-A7 dLOSS/dtheta by reverse mode (u-adjoint 2 A(alpha) q, MLP backward, reduction)
 *   A8 Adam step ("Adam optimizer")
 *
 * alpha_ij = K_ij ((1 - S_ij) + M S_ij), M = mu_w/mu_g (Eq. 23 first line, PAPER.md:369,
 * non-dimensional reading R10), and b = h^2 f with f the right side of -div(alpha grad p) = f
 * (reading R1; for an injection well f > 0). All readings are listed in DESIGN.md §2.
 *
 * Conventions (apply to every entry point):
 *  - N is the number of grid intervals per axis, h = 1/N, nodes (x_i, y_j) = (i/N, j/N),
 *    0 <= i,j <= N (Eq. 21, reading R9). Unknowns are the (N-1)^2 interior nodes.
 *  - Host fields are float32, row-major (N+1) x (N+1): F[j*(N+1) + i] at (x_i, y_j).
 *  - theta is float32, flattened W1 (row-major out x in), b1, W2, b2, ..., W_{L+1}, b_{L+1}.
 *  - All pointer arguments are caller-owned; inputs are copied before the call returns
 *    (unless documented as device pointers), outputs are written into caller buffers.
 *  - A context owns all of its device memory, its CUDA stream (or uses the one given in
 *    opts.stream) and its captured CUDA graphs. A context is NOT thread-safe; several
 *    contexts may coexist (one per GPU / per independent problem).
 *  - Return value: CRVPINN_OK (0) or a negative code; crvpinn_last_error() explains it.
 *  - The library never falls back to a CPU path: without a usable sm_100 device every
 *    call that needs one returns CRVPINN_ECUDA.
 */
#ifndef CRVPINN_H
#define CRVPINN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct crvpinn_ctx crvpinn_ctx;   /* opaque */

enum {
    CRVPINN_OK = 0,
    CRVPINN_EINVAL = -1,      /* bad argument: N, widths, null required pointer, n < 1 */
    CRVPINN_ENOMEM = -2,      /* device allocation failed */
    CRVPINN_ECUDA = -3,       /* CUDA runtime error / no sm_100 device */
    CRVPINN_ENONFINITE = -4,  /* loss or gradient became non-finite; theta restored */
    CRVPINN_EDOMAIN = -5      /* K <= 0 or a non-finite input field */
};

/* Arithmetic of the MLP contractions (A1, A6). The stencil, Gram solve, reductions and
 * Adam are fp32 (reductions of the loss in fp64) in every mode. */
enum {
    CRVPINN_PREC_TENSOR = 0,  /* tcgen05 tensor cores, fp16 operands (10-bit mantissa, same as
                                 TF32): forward activations split hi+lo (2 MMAs), backward 1 MMA
                                 with power-of-two gradient scaling; fp32 accumulate in TMEM.
                                 Parity class: north_star's "TF32" tolerances. */
    CRVPINN_PREC_FP32 = 1     /* SIMT FFMA fp32 everywhere. Parity class: "fp32" tolerances. */
};

typedef struct {
    double lr;              /* Adam learning rate (default 1e-3, BASELINE.json configs[0]) */
    double beta1, beta2;    /* default 0.9, 0.999 (reading R7) */
    double eps;             /* default 1e-8 */
    double mobility_ratio;  /* M = mu_w/mu_g, default 25.35/3.95 (Table 1) */
    int precision;          /* CRVPINN_PREC_*, default CRVPINN_PREC_TENSOR */
    uint64_t seed;          /* Xavier init seed when theta0 == NULL */
    void *stream;           /* cudaStream_t to run on; NULL = the context creates its own */
    int device;             /* CUDA device ordinal, default 0 */
    /* Gravity term of Eq. 23's RHS, grad+ . (g K ((1-S) rho_w/mu_w + S rho_g/mu_g)) (PAPER.md:370,
     * SURVEY.md §8(f) f1), read non-dimensionally (R23): g = -gravity * y-hat and
     * beta = (1-S) + M (rho_g/rho_w) S, so b_kl = h^2 f_kl + h gravity (gamma_{k,l+1} - gamma_{k,l}),
     * gamma = K beta. Recomputed with alpha on every set_saturation. */
    double gravity;         /* non-dimensional gravity number, default 0 (the configs have none, R11) */
    double density_ratio;   /* rho_g/rho_w, default 479/1045 (Table 1) */
    /* Point sharding across GPUs. The MLP points (the
     * set the loss sums over) split into shard_world contiguous ranges of
     * 128-point tiles (crvpinn_shard_tiles); this context runs the forward and backward of range
     * shard_rank only. One Adam iteration then exchanges twice: an all-reduce (sum) of the
     * lattice field u after the forward (each shard writes its own points into a zeroed field,
     * so the sum is the whole field exactly), and an all-reduce (sum) of the gradient after the
     * backward. Stencil, Gram solve, loss and Adam run replicated on every shard. Tensor path
     * only. Default shard_rank 0, shard_world 1 (unsharded). */
    int shard_rank;
    int shard_world;
    /* nccl = 1: the context creates an NCCL communicator (rank shard_rank of shard_world) from
     * nccl_id (crvpinn_nccl_unique_id on one rank, shared by the caller) and issues the two
     * all-reduces inside every iteration (and inside the captured graphs). Allowed at
     * shard_world 1. nccl = 0 with shard_world > 1: the caller exchanges, using
     * crvpinn_shard_forward / crvpinn_shard_backward; crvpinn_step and crvpinn_loss_grad then
     * fail with EINVAL. libnccl.so.2 is loaded on first use (dlopen), not at library load.
     * θ, the Adam state and the fields are replicated: every rank of a group must make the same
     * calls with the same arguments (create, set_saturation, step, set_params, set_adam), and
     * crvpinn_step / crvpinn_loss_grad / crvpinn_eval are collective (each rank calls them once,
     * in the same order). */
    int nccl;
    unsigned char nccl_id[128];
} crvpinn_opts;

/* Fill *o with the defaults listed above. */
void crvpinn_default_opts(crvpinn_opts *o);

/* Create a problem on grid N (power of two, 16 <= N <= 2048) with layer widths
 * widths[0..n_widths-1] = {2, w, ..., w, 1} (hidden widths multiples of 32, <= 256, at most
 * 16 layers). CRVPINN_PREC_TENSOR further requires (else EINVAL): at least two hidden layers
 * (one hidden-to-hidden GEMM), all hidden widths equal, and w in {32, 64, 96, 128, 224, 256}
 * (w is zero-padded to WP = 64 ceil(w/64) in {64, 128, 256}; WP = 192, i.e. w = 160 or 192, has
 * no kernel instantiation). CRVPINN_PREC_FP32 takes every width set above.
 * K, S, f: host (N+1)^2 float32 fields (K > 0; S is clamped to [0,1]).
 * theta0: host float32 of crvpinn_num_params entries, or NULL for Xavier-uniform (biases 0).
 * Runs step A0 (alpha, b) and builds the Gram-solve constants (Eq. 28 "factorization performed
 * only once", realised as the sine basis of G). Adam state starts at zero. */
int crvpinn_create(crvpinn_ctx **out, int N, int n_widths, const int *widths,
                   const float *K, const float *S, const float *f,
                   const float *theta0, const crvpinn_opts *opts);

/* Replace the saturation field (host, (N+1)^2) and recompute alpha (step A0).
 * PAPER.md:447-452 (§6 step 7: "including the actual saturation S_g^n"). */
int crvpinn_set_saturation(crvpinn_ctx *ctx, const float *S);

/* Same, with S a DEVICE pointer (float32, (N+1)^2) on the context's device; the copy is
 * stream-ordered on the context stream. Used when the saturation is already resident. */
int crvpinn_set_saturation_device(crvpinn_ctx *ctx, const void *S_dev);

/* Pretraining: n_iters Adam iterations on the current fields (§6 step 2).
 * loss_hist (nullable, n_iters doubles): loss_hist[k] = LOSS(theta_k) before update k+1. */
int crvpinn_pretrain(crvpinn_ctx *ctx, int n_iters, double *loss_hist);

/* One pressure update: n_adam Adam iterations (§6 step 7; 100 in the paper).
 * Same semantics as crvpinn_pretrain; theta and the Adam state (m, v, t) persist across calls
 * (reading R8). All n_adam iterations run as one CUDA graph (captured on first use per n).
 * On a non-finite loss/gradient returns CRVPINN_ENONFINITE and restores theta and the Adam
 * state to their values at call entry. */
int crvpinn_step(crvpinn_ctx *ctx, int n_adam, double *loss_hist);

/* Evaluate the network on the lattice: p_out (host, (N+1)^2 float32) = PINN_ij, exactly 0 on
 * the boundary (the hand-off to the IGA projection). */
int crvpinn_eval(crvpinn_ctx *ctx, float *p_out);

/* Continuous evaluation of the trained network with its hard cutoff at arbitrary points,
 * p(x, y) = 16 x(1-x) y(1-y) net_theta(x, y), as the IGA L2 projection needs it at
 * quadrature points (§6 step 4), in the
 * context's precision mode (same kernels as the lattice forward). xy: host float32 [n][2] pairs
 * (x, y); p_out: host float32 [n]. n == 0 is a no-op. EINVAL: n < 0 or a null pointer with n > 0;
 * EDOMAIN: a non-finite coordinate (nothing is written). Synchronising. */
int crvpinn_eval_points(crvpinn_ctx *ctx, long n, const float *xy, float *p_out);

/* the discrete system A(alpha) u = b itself -- the reference pressure the
 * paper gets from MUMPS -- for the context's current alpha and b (K, S, f,
 * gravity), solved on the GPU by conjugate gradients preconditioned with the exact Gram solve
 * G^-1 of Eq. 26/28 (spectrally equivalent to A(alpha)), fp32 vectors, fp64
 * dot products, starting from u = 0. Stops when ||r|| / ||b|| <= rtol (checked every 20
 * iterations) or after max_iter iterations. u_out: host (N+1)^2 float32, boundary 0 (nullable);
 * iters, rel_res (nullable): iterations used and the TRUE relative residual ||b - A u|| / ||b||
 * of the returned u (fp64). EINVAL: rtol <= 0 or max_iter < 1; ENONFINITE: non-finite residual.
 * Returns CRVPINN_OK also when rtol was not reached (check rel_res). Does not touch theta. */
int crvpinn_direct_solve(crvpinn_ctx *ctx, double rtol, int max_iter, float *u_out, int *iters, double *rel_res);

/* LOSS (Eq. 27) and dLOSS/dtheta at the current theta, no update. grad nullable. */
int crvpinn_loss_grad(crvpinn_ctx *ctx, double *loss, float *grad);

/* Intermediates of the last crvpinn_loss_grad (test hook, host float32; each nullable):
 * u (N+1)^2 lattice, res (N-1)^2, q (N-1)^2, gu (N+1)^2 lattice = dLOSS/du (0 on boundary).
 * On a sharded context without a communicator (caller exchange) they are those of the last
 * crvpinn_shard_forward / _backward: u as this rank's forward left it (its own points only)
 * unless _backward has since received the summed u. Never fails on a valid ctx. */
int crvpinn_get_intermediates(crvpinn_ctx *ctx, float *u, float *res, float *q, float *gu);

size_t crvpinn_num_params(const crvpinn_ctx *ctx);

/* theta (float32, num_params). get is stream-ordered and synchronising. */
int crvpinn_get_params(crvpinn_ctx *ctx, float *theta);
int crvpinn_set_params(crvpinn_ctx *ctx, const float *theta);

/* Checkpoint / resume of the Adam state (m, v: float32 num_params each; t: step count). */
int crvpinn_get_adam(crvpinn_ctx *ctx, float *m, float *v, int64_t *t);
int crvpinn_set_adam(crvpinn_ctx *ctx, const float *m, const float *v, int64_t t);

/* Per-stage device timing of the iterations run by crvpinn_step while profiling is on:
 * CUDA events recorded on the context stream around each stage INSIDE the captured graph.
 * Stages: 0 = MLP forward (A1), 1 = stencil + Gram + loss + adjoint (A2-A5),
 * 2 = MLP backward + weight-gradient reduction (A6-A7), 3 = Adam (A8).
 * Enabling/disabling drops cached graphs. ms_sum[s] accumulates milliseconds over all
 * profiled iterations since the last reset; *n_iters receives their count. */
int crvpinn_set_profiling(crvpinn_ctx *ctx, int on);
int crvpinn_get_profile(crvpinn_ctx *ctx, double *ms_sum /* [4] */, int64_t *n_iters, int reset);

/* Number of kernel launches one Adam iteration issues (for the bench's gpu_launches). */
int crvpinn_launches_per_iter(const crvpinn_ctx *ctx);

/* Context stream (cudaStream_t) for callers that synchronise with it. */
void *crvpinn_stream(const crvpinn_ctx *ctx);

const char *crvpinn_last_error(const crvpinn_ctx *ctx);   /* ctx may be NULL (global error) */

void crvpinn_destroy(crvpinn_ctx *ctx);

/* ------------------------------------------------------------ point sharding (f4) */
/* Shard r of w over an N x N point set: tiles [*tile0, *tile0 + *ntiles) of T = N*N/128, the
 * balanced split tile0 = floor(r T / w) (shards differ by at most one tile). Pure host
 * arithmetic (no device needed). EINVAL unless N is a power of two in [16, 2048] and
 * 0 <= r < w <= T. */
int crvpinn_shard_tiles(int N, int rank, int world, long *tile0, long *ntiles);

/* A fresh NCCL unique id (ncclGetUniqueId) for opts.nccl_id, to be created on one rank and sent
 * to the others by the caller. ECUDA if libnccl.so.2 cannot be loaded. */
int crvpinn_nccl_unique_id(unsigned char id[128]);

/* The two halves of one iteration around the exchange, for callers that move the data
 * themselves (and for single-GPU tests of a sharded decomposition). No collective is issued.
 * shard_forward: u_part (host, (N+1)^2 floats) = this shard's points of u = cutoff * net, zero
 * at every other node. shard_backward: given the whole field u_full (host, the sum of every
 * shard's u_part), runs A2-A5 (replicated) and the backward of this shard's points: *loss = the
 * loss of u_full, grad_part (host, num_params floats) = this shard's share of dLOSS/dtheta
 * (the gradient is the sum of the shares). theta and the Adam state do not change. */
int crvpinn_shard_forward(crvpinn_ctx *ctx, float *u_part);
int crvpinn_shard_backward(crvpinn_ctx *ctx, const float *u_full, double *loss, float *grad_part);

/* ========================================================================== IGA-ADS (f3)
 * the explicit saturation step of IGA-ADS on the GPU (§3-§4), the
 * second half of the hybrid loop (§6 step 5 / §7). A crvpinn_iga is one tensor-product spline
 * space on [0,1]^2: B-splines of degree r (C^{r-1}, Eq. 11) on open uniform
 * knots with ne elements per axis, nb = ne + r functions per axis, Gauss-Legendre with r+1 points
 * per element and axis (reading R27). Coefficient matrices are host float32 [nb][nb] indexed
 * [l][k] (row = y basis index, column = x basis index); element fields [ne][ne] are [ey][ex].
 * All calls are synchronous, take host buffers and return CRVPINN_* codes. */
typedef struct crvpinn_iga crvpinn_iga;

/* ne in [1, 8192], 1 <= degree <= 6. EINVAL on bad sizes, ECUDA without a device. */
int crvpinn_iga_create(crvpinn_iga **out, int n_elements, int degree, int device);
int crvpinn_iga_num_basis(const crvpinn_iga *g);            /* nb (per axis) */
long crvpinn_iga_num_quad_points(const crvpinn_iga *g);     /* (ne (r+1))^2 */

/* Tensor Gauss points, x fastest: xy[2p], xy[2p+1] for p = (ey(r+1)+qy) ne(r+1) + ex(r+1) + qx. */
int crvpinn_iga_quad_points(crvpinn_iga *g, float *xy);

/* Isogeometric L2 projection (Eq. 12-14): coef = (M^x (x) M^y)^-1 L, L_kl = (f, B_k B_l) by the
 * tensor Gauss rule from f's values fq at the quadrature points (order of crvpinn_iga_quad_points;
 * e.g. the CRVPINN pressure from crvpinn_eval_points, §6 step 4). The mass solve runs direction by
 * direction with banded LDL^T factors (bandwidth r; the paper's Thomas algorithm). */
int crvpinn_iga_project(crvpinn_iga *g, const float *fq, float *coef);

/* One explicit step of Eq. 10 (readings R24-R26):
 *   (S_out, v) = (S, v) + (tau/phi) ( -M S K (grad p . grad v + r Gr v_y) + q v )  for all v,
 * then the boundary coefficients of S_out are set to 0 (zero Dirichlet saturation).
 * S, P: coefficients of S^n and p^n; K_elem, q_elem: per-element permeability and gas source;
 * M = mobility_ratio (mu_w/mu_g), r = density_ratio (rho_g/rho_w), Gr = gravity (R23). EINVAL:
 * tau < 0, phi <= 0, non-finite parameters or null pointers. */
int crvpinn_iga_saturation_step(crvpinn_iga *g, const float *S, const float *P, const float *K_elem,
                                const float *q_elem, double tau, double phi, double mobility_ratio,
                                double density_ratio, double gravity, float *S_out);

/* Field value (and gradient, nullable: [n][2]) of coef at n points (clamped to [0,1]^2), e.g. the
 * saturation at the CRVPINN collocation lattice (§6 step 7). */
int crvpinn_iga_eval(crvpinn_iga *g, const float *coef, long n, const float *xy, float *val, float *grad);

double crvpinn_iga_last_ms(const crvpinn_iga *g);   /* device time of the last project / step (ms) */
const char *crvpinn_iga_last_error(const crvpinn_iga *g);
void crvpinn_iga_destroy(crvpinn_iga *g);

#ifdef __cplusplus
}
#endif
#endif /* CRVPINN_H */
