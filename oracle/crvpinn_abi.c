/*
 * crvpinn_abi.c -- the fp64 CPU ORACLE behind the product's C ABI.
 *
 * TEST INFRASTRUCTURE ONLY (like crvpinn_oracle.c): loaded by tests/ for ABI-level A/B runs, in
 * which one ctypes driver calls the same entry points of this library and of the CUDA library
 * (paper_2604_20731_b200/libcrvpinn.so) on the same inputs. Nothing here is shared with the
 * product: the prototypes and the options layout below are restated from the ABI's documented
 * contract (include/crvpinn.h is NOT included), and every computation is an orc_* call of
 * crvpinn_oracle.c, i.e. the paper's algorithm step by step in fp64.
 *
 * Core calls of §8(b) (north_star: crvpinn_create(grid, layer widths, K field, S field, source),
 * crvpinn_pretrain(n), crvpinn_step(n_adam), crvpinn_eval(p_out)) and the parity hooks:
 *   crvpinn_default_opts, crvpinn_create, crvpinn_set_saturation, crvpinn_pretrain, crvpinn_step,
 *   crvpinn_eval, crvpinn_loss_grad, crvpinn_get_intermediates, crvpinn_num_params,
 *   crvpinn_get_params, crvpinn_set_params, crvpinn_get_adam, crvpinn_last_error, crvpinn_destroy.
 * Differences from the product, by design: theta0 must be given (the product's seeded Xavier
 * draw is not restated; NULL -> EINVAL); precision, stream, device and the sharding fields are
 * ignored (fp64 on the host); state is fp64 and converted to float32 at the boundary.
 * Error codes: OK 0, EINVAL -1, ENOMEM -2, ENONFINITE -4 (theta and the Adam state restored to
 * their values at call entry, §6 / SPEC.md:438), EDOMAIN -5 (K <= 0 or non-finite field).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- the oracle (crvpinn_oracle.c) */
typedef struct orc_ctx orc_ctx;
orc_ctx *orc_create(int N, int nl, const int *widths, const float *K, const float *S, const float *f,
                    const float *theta0, double mobility, double lr, double beta1, double beta2, double eps,
                    int factor_gram, double gravity, double rho_ratio);
void orc_destroy(orc_ctx *c);
long orc_num_params(const orc_ctx *c);
void orc_get_theta(const orc_ctx *c, double *th);
void orc_set_theta(orc_ctx *c, const double *th);
void orc_get_adam(const orc_ctx *c, double *m, double *v, long *t);
void orc_set_adam(orc_ctx *c, const double *m, const double *v, long t);
int orc_set_saturation(orc_ctx *c, const float *K, const float *S);
void orc_forward(const orc_ctx *c, const double *th, double *u);
double orc_loss_grad(const orc_ctx *c, const double *th_in, double *grad, double *u_out, double *res_out,
                     double *q_out, double *gu_out);
void orc_adam_step(orc_ctx *c, const double *g);

/* ---- the ABI's options record, restated from its documented layout */
typedef struct {
    double lr, beta1, beta2, eps, mobility_ratio;
    int precision;
    uint64_t seed;
    void *stream;
    int device;
    double gravity, density_ratio;
    int shard_rank, shard_world, nccl;
    unsigned char nccl_id[128];
} abi_opts;

typedef struct {
    orc_ctx *o;
    int N;
    float *K;                 /* kept for set_saturation (alpha and the gravity term need K) */
    double *m0, *v0, *th0;    /* call-entry snapshot for the ENONFINITE restore */
    long t0;
    char err[256];
} abi_ctx;

static char g_err[256] = "";

static int fail(abi_ctx *c, int code, const char *msg) {
    char *dst = c ? c->err : g_err;
    strncpy(dst, msg, 255);
    dst[255] = 0;
    return code;
}

void crvpinn_default_opts(abi_opts *o) {
    memset(o, 0, sizeof(*o));
    o->lr = 1e-3;
    o->beta1 = 0.9;
    o->beta2 = 0.999;
    o->eps = 1e-8;
    o->mobility_ratio = 25.35 / 3.95;     /* Table 1 */
    o->density_ratio = 479.0 / 1045.0;    /* Table 1 */
    o->shard_world = 1;
}

static int fields_ok(const float *a, long n, int positive) {
    for (long i = 0; i < n; ++i)
        if (!isfinite(a[i]) || (positive && !(a[i] > 0.0f))) return 0;
    return 1;
}

int crvpinn_create(abi_ctx **out, int N, int n_widths, const int *widths, const float *K, const float *S,
                   const float *f, const float *theta0, const abi_opts *opts) {
    if (!out || !widths || !K || !S || !f) return fail(NULL, -1, "null argument");
    *out = NULL;
    if (N < 2 || (N & (N - 1)) != 0 || n_widths < 3 || n_widths > 17 || widths[0] != 2 || widths[n_widths - 1] != 1)
        return fail(NULL, -1, "bad grid or widths");
    if (!theta0) return fail(NULL, -1, "the oracle ABI needs theta0 (no Xavier draw)");
    const long nn = (long)(N + 1) * (N + 1);
    if (!fields_ok(K, nn, 1) || !fields_ok(S, nn, 0) || !fields_ok(f, nn, 0)) return fail(NULL, -5, "bad field");
    abi_opts d;
    crvpinn_default_opts(&d);
    if (!opts) opts = &d;
    abi_ctx *c = (abi_ctx *)calloc(1, sizeof(abi_ctx));
    if (!c) return fail(NULL, -2, "out of host memory");
    c->N = N;
    c->o = orc_create(N, n_widths - 1, widths, K, S, f, theta0, opts->mobility_ratio, opts->lr, opts->beta1,
                      opts->beta2, opts->eps, 1, opts->gravity, opts->density_ratio);
    c->K = (float *)malloc(sizeof(float) * nn);
    if (!c->o || !c->K) {
        orc_destroy(c->o);
        free(c->K);
        free(c);
        return fail(NULL, -2, "oracle allocation failed");
    }
    memcpy(c->K, K, sizeof(float) * nn);
    const long np = orc_num_params(c->o);
    c->m0 = (double *)malloc(sizeof(double) * np);
    c->v0 = (double *)malloc(sizeof(double) * np);
    c->th0 = (double *)malloc(sizeof(double) * np);
    *out = c;
    return 0;
}

int crvpinn_set_saturation(abi_ctx *c, const float *S) {
    if (!c || !S) return fail(c, -1, "null argument");
    if (!fields_ok(S, (long)(c->N + 1) * (c->N + 1), 0)) return fail(c, -5, "non-finite S");
    orc_set_saturation(c->o, c->K, S);   /* A0 (step 7 on the current S) */
    return 0;
}

/* n Adam iterations; hist[k] = LOSS before update k+1 */
static int run(abi_ctx *c, int n, double *hist) {
    if (!c || n < 1) return fail(c, -1, "bad argument");
    const long np = orc_num_params(c->o);
    orc_get_theta(c->o, c->th0);
    orc_get_adam(c->o, c->m0, c->v0, &c->t0);
    double *g = (double *)malloc(sizeof(double) * np);
    if (!g) return fail(c, -2, "out of host memory");
    for (int k = 0; k < n; ++k) {
        const double loss = orc_loss_grad(c->o, NULL, g, NULL, NULL, NULL, NULL);
        if (hist) hist[k] = loss;
        int finite = isfinite(loss);
        for (long i = 0; i < np && finite; ++i) finite = isfinite(g[i]);
        if (!finite) {
            orc_set_theta(c->o, c->th0);   /* the ABI contract: theta and Adam state at call entry */
            orc_set_adam(c->o, c->m0, c->v0, c->t0);
            free(g);
            return fail(c, -4, "non-finite loss or gradient");
        }
        orc_adam_step(c->o, g);
    }
    free(g);
    return 0;
}

int crvpinn_pretrain(abi_ctx *c, int n_iters, double *loss_hist) { return run(c, n_iters, loss_hist); }
int crvpinn_step(abi_ctx *c, int n_adam, double *loss_hist) { return run(c, n_adam, loss_hist); }

int crvpinn_eval(abi_ctx *c, float *p_out) {
    if (!c || !p_out) return fail(c, -1, "null argument");
    const long nn = (long)(c->N + 1) * (c->N + 1);
    double *u = (double *)malloc(sizeof(double) * nn);
    if (!u) return fail(c, -2, "out of host memory");
    orc_get_theta(c->o, c->th0);
    orc_forward(c->o, c->th0, u);
    for (long i = 0; i < nn; ++i) p_out[i] = (float)u[i];
    free(u);
    return 0;
}

int crvpinn_loss_grad(abi_ctx *c, double *loss, float *grad) {
    if (!c || !loss) return fail(c, -1, "null argument");
    const long np = orc_num_params(c->o);
    double *g = (double *)malloc(sizeof(double) * np);
    if (!g) return fail(c, -2, "out of host memory");
    *loss = orc_loss_grad(c->o, NULL, g, NULL, NULL, NULL, NULL);
    if (grad)
        for (long i = 0; i < np; ++i) grad[i] = (float)g[i];
    free(g);
    return isfinite(*loss) ? 0 : fail(c, -4, "non-finite loss");
}

int crvpinn_get_intermediates(abi_ctx *c, float *u, float *res, float *q, float *gu) {
    if (!c) return fail(c, -1, "null ctx");
    const long nn = (long)(c->N + 1) * (c->N + 1), n2 = (long)(c->N - 1) * (c->N - 1);
    double *du = (double *)malloc(sizeof(double) * nn), *dgu = (double *)malloc(sizeof(double) * nn);
    double *dr = (double *)malloc(sizeof(double) * n2), *dq = (double *)malloc(sizeof(double) * n2);
    if (!du || !dgu || !dr || !dq) {
        free(du); free(dgu); free(dr); free(dq);
        return fail(c, -2, "out of host memory");
    }
    orc_loss_grad(c->o, NULL, NULL, du, dr, dq, dgu);
    for (long i = 0; i < nn; ++i) {
        if (u) u[i] = (float)du[i];
        if (gu) gu[i] = (float)dgu[i];
    }
    for (long i = 0; i < n2; ++i) {
        if (res) res[i] = (float)dr[i];
        if (q) q[i] = (float)dq[i];
    }
    free(du); free(dgu); free(dr); free(dq);
    return 0;
}

size_t crvpinn_num_params(const abi_ctx *c) { return c ? (size_t)orc_num_params(c->o) : 0; }

int crvpinn_get_params(abi_ctx *c, float *theta) {
    if (!c || !theta) return fail(c, -1, "null argument");
    const long np = orc_num_params(c->o);
    orc_get_theta(c->o, c->th0);
    for (long i = 0; i < np; ++i) theta[i] = (float)c->th0[i];
    return 0;
}

int crvpinn_set_params(abi_ctx *c, const float *theta) {
    if (!c || !theta) return fail(c, -1, "null argument");
    const long np = orc_num_params(c->o);
    for (long i = 0; i < np; ++i) c->th0[i] = (double)theta[i];
    orc_set_theta(c->o, c->th0);
    return 0;
}

int crvpinn_get_adam(abi_ctx *c, float *m, float *v, int64_t *t) {
    if (!c) return fail(c, -1, "null ctx");
    const long np = orc_num_params(c->o);
    long tt = 0;
    orc_get_adam(c->o, c->m0, c->v0, &tt);
    for (long i = 0; i < np; ++i) {
        if (m) m[i] = (float)c->m0[i];
        if (v) v[i] = (float)c->v0[i];
    }
    if (t) *t = (int64_t)tt;
    return 0;
}

const char *crvpinn_last_error(const abi_ctx *c) { return c ? c->err : g_err; }

void crvpinn_destroy(abi_ctx *c) {
    if (!c) return;
    orc_destroy(c->o);
    free(c->K); free(c->m0); free(c->v0); free(c->th0);
    free(c);
}
