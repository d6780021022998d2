/*
 * crvpinn_oracle.c -- plain, slow, fp64 CPU ORACLE of the CRVPINN pressure update.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library. The product path (the CUDA
 * library under paper_2604_20731_b200/) shares no code, header, table or helper with it.
 *
 * What it computes, step by step in the paper's order (§5-§6, arXiv 2604.20731):
 *   A0  alpha_ij = ((1-S_ij)/mu_w + S_ij/mu_g) K_ij      PAPER.md:369 (Eq. 23), read
 *       non-dimensionally as K((1-S) + M S), M = mu_w/mu_g (reading R10);
 *       b_kl = h^2 f_kl, f the right side of -div(alpha grad p) = f (reading R1). With the
 *       gravity term of Eq. 23's RHS (reading R23) the right
 *       side is f - grad+ . F, F_ij = g K_ij ((1-S_ij) + M r S_ij), g = (0, -gravity),
 *       r = rho_g/rho_w, grad+ . F = forward differences of Eq. 22.
 *   eval_points: p(x,y) = cutoff(x,y) net_theta(x,y) at arbitrary points.
 *   A1  PINN_ij = 16 x(1-x) y(1-y) * net_theta(x_i, y_j), tanh MLP
 *       (architecture/cutoff: readings R5, R6).
 *   A2  RES_kl = (alpha grad+ PINN, grad+ delta_kl)_h - (RHS, delta_kl)_h   Eq. 25,
 *       PAPER.md:378-381, with (u,v)_h = h^2 sum_p u(p)v(p) and grad+ of
 *       Eq. 22. The sum over p is written out over the three nodes where
 *       grad+ delta_kl is non-zero: p=(k,l): (-1/h,-1/h); p=(k-1,l): (1/h,0); p=(k,l-1): (0,1/h).
 *   A3  G = h^-2 (4 on the diagonal, -1 for the 4 neighbours)   Eq. 26, PAPER.md:398-406,
 *       LU-factorised ONCE (Eq. 28), then forward/back substitution.
 *       Banded Doolittle LU without pivoting (G is SPD and diagonally dominant) in the
 *       natural row-major order r = (l-1) n + (k-1); since G is symmetric, L_ik = U_ki/U_kk
 *       so only the upper band of U is stored. Eq. 28 writes "U z = RES, L q = z"; the
 *       consistent order L z = RES, U q = z is used (reading R19).
 *   A4  LOSS = RES^T q = RES^T G^-1 RES   Eq. 27.
 *   A5  dLOSS/du_p = sum_kl 2 q_kl dRES_kl/du_p (reverse mode through the literal residual).
 *   A6  reverse-mode through the cutoff and the MLP, per point, fp64, fixed-order reduction.
 *   A8  Adam (Kingma & Ba; "Adam optimizer"), beta1/beta2/eps = reading R7.
 *
 * Parity pins for every function live in tests/test_oracle_pins.py (P1..P13).
 * Build: gcc -O2 -fopenmp -shared -fPIC (see __graft_entry__.build()).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_LAYERS 16

typedef struct orc_ctx {
    int N, n;                  /* intervals per axis; n = N-1 unknowns per axis */
    double h;
    int nl;                    /* number of weight layers (hidden + output) */
    int widths[ORC_MAX_LAYERS + 1];
    long np;                   /* parameter count */
    long woff[ORC_MAX_LAYERS], boff[ORC_MAX_LAYERS];
    double mobility;
    double gravity, rho_ratio; /* gravity number and rho_g/rho_w (reading R23) */
    double *alpha;             /* (N+1)^2 nodes, [j*(N+1)+i] */
    double *f;                 /* (N+1)^2 nodes: the source f as given */
    double *b;                 /* (N+1)^2 nodes: h^2 (f - grad+ . F) */
    double *U;                 /* band LU of G: n^2 rows x (n+1): U[r*(n+1)+d] = U(r, r+d) */
    double *theta, *m, *v;     /* parameters and Adam moments */
    long t;                    /* Adam step counter */
    double lr, beta1, beta2, eps;
} orc_ctx;

static long idx(const orc_ctx *c, int i, int j) { return (long)j * (c->N + 1) + i; }

/* ---------------------------------------------------------------- A0: alpha and b */
static void set_alpha(orc_ctx *c, const float *K, const float *S) {
    long nn = (long)(c->N + 1) * (c->N + 1);
    for (long p = 0; p < nn; ++p) {
        double s = (double)S[p];
        if (s < 0.0) s = 0.0;          /* S clamped to [0,1] (reading R10) */
        if (s > 1.0) s = 1.0;
        c->alpha[p] = (double)K[p] * ((1.0 - s) + c->mobility * s);
    }
}

/* b = h^2 (f - grad+ . F): (RHS, delta_kl)_h of Eq. 24-25 with the sign of reading R1. F is the
 * node field g K beta with g = (0, -gravity) and beta = (1-S) + M r S (non-dimensional form of
 * (1-S) rho_w/mu_w + S rho_g/mu_g, divided by rho_w/mu_w); its x-component is zero. */
static void set_rhs(orc_ctx *c, const float *K, const float *S) {
    int N = c->N;
    long nn = (long)(N + 1) * (N + 1);
    double h = c->h;
    double *Fx = (double *)calloc(nn, sizeof(double)), *Fy = (double *)calloc(nn, sizeof(double));
    for (long p = 0; p < nn; ++p) {
        double s = (double)S[p];
        if (s < 0.0) s = 0.0;
        if (s > 1.0) s = 1.0;
        double beta = (1.0 - s) + c->mobility * c->rho_ratio * s;
        Fx[p] = 0.0 * (double)K[p] * beta;              /* g_x = 0 */
        Fy[p] = -c->gravity * (double)K[p] * beta;     /* g_y = -gravity */
    }
    for (int j = 0; j <= N; ++j)
        for (int i = 0; i <= N; ++i) {
            double div = 0.0;   /* grad+ . F at (i, j); defined where (i+1, j) and (i, j+1) exist */
            if (i < N && j < N)
                div = (Fx[idx(c, i + 1, j)] - Fx[idx(c, i, j)]) / h + (Fy[idx(c, i, j + 1)] - Fy[idx(c, i, j)]) / h;
            c->b[idx(c, i, j)] = h * h * (c->f[idx(c, i, j)] - div);
        }
    free(Fx);
    free(Fy);
}

int orc_set_saturation(orc_ctx *c, const float *K, const float *S) {
    set_alpha(c, K, S);
    set_rhs(c, K, S);
    return 0;
}

void orc_get_b(const orc_ctx *c, double *out) {
    memcpy(out, c->b, sizeof(double) * (long)(c->N + 1) * (c->N + 1));
}

/* ---------------------------------------------------------------- f2: the discrete system itself */
/* solve A(alpha) u = b directly -- the reference pressure the paper obtains
 * with MUMPS. A(alpha) is read off the residual of Eq. 25 (RES = A u - b, stencil
 * of A2 / reading R16): row (k,l) has diagonal alpha_{k-1,l} + alpha_{k,l-1} + 2 alpha_{k,l} and
 * -alpha_{k-1,l}, -alpha_{k,l-1}, -alpha_{k,l}, -alpha_{k,l} for the neighbours (k-1,l), (k,l-1),
 * (k+1,l), (k,l+1) (boundary neighbours drop out: u = 0 there). A is symmetric; it is factorised
 * by banded Doolittle LU (half-bandwidth n, natural row-major order) and solved by forward/back
 * substitution. u_out: (N+1)^2 lattice, boundary 0. Returns 0, or -1 on allocation failure. */
int orc_direct_solve(const orc_ctx *c, double *u_out) {
    int N = c->N, n = c->n;
    long n2 = (long)n * n, bw = n + 1;
    double *U = (double *)calloc((size_t)n2 * bw, sizeof(double));
    double *z = (double *)malloc(sizeof(double) * n2);
    if (!U || !z) { free(U); free(z); return -1; }
    for (int l = 1; l <= n; ++l)
        for (int k = 1; k <= n; ++k) {
            long r = (long)(l - 1) * n + (k - 1);
            U[r * bw + 0] = c->alpha[idx(c, k - 1, l)] + c->alpha[idx(c, k, l - 1)] + 2.0 * c->alpha[idx(c, k, l)];
            if (k < n) U[r * bw + 1] = -c->alpha[idx(c, k, l)];   /* (k+1, l) */
            if (l < n) U[r * bw + n] = -c->alpha[idx(c, k, l)];   /* (k, l+1) */
        }
    for (long k = 0; k < n2; ++k) {
        const double *uk = U + k * bw;
        long iend = k + n < n2 - 1 ? k + n : n2 - 1;
#pragma omp parallel for schedule(static) if (n >= 48)
        for (long i = k + 1; i <= iend; ++i) {
            double lik = uk[i - k] / uk[0];   /* A symmetric: A(i,k) = U(k,i) before row k is used */
            if (lik == 0.0) continue;
            double *ui = U + i * bw;
            for (long j = i; j <= iend; ++j) ui[j - i] -= lik * uk[j - k];
        }
    }
    /* forward: L z = b (L_ik = U(k,i)/U(k,k)), backward: U u = z */
    for (long i = 0; i < n2; ++i) {
        int l = (int)(i / n) + 1, k = (int)(i % n) + 1;
        double v = c->b[idx(c, k, l)];
        long kbeg = i - n > 0 ? i - n : 0;
        for (long kk = kbeg; kk < i; ++kk) v -= U[kk * bw + (i - kk)] / U[kk * bw] * z[kk];
        z[i] = v;
    }
    long nn = (long)(N + 1) * (N + 1);
    for (long p = 0; p < nn; ++p) u_out[p] = 0.0;
    for (long i = n2 - 1; i >= 0; --i) {
        double v = z[i];
        long jend = i + n < n2 - 1 ? i + n : n2 - 1;
        for (long j = i + 1; j <= jend; ++j) {
            int lj = (int)(j / n) + 1, kj = (int)(j % n) + 1;
            v -= U[i * bw + (j - i)] * u_out[idx(c, kj, lj)];
        }
        int l = (int)(i / n) + 1, k = (int)(i % n) + 1;
        u_out[idx(c, k, l)] = v / U[i * bw];
    }
    free(U);
    free(z);
    return 0;
}

/* ---------------------------------------------------------------- A3: factor G once */
/* Entry (r, r+d) of G (Eq. 26) for d >= 0, r = (l-1) n + (k-1). */
static double gram_entry(const orc_ctx *c, long r, long d) {
    int n = c->n;
    double h2i = 1.0 / (c->h * c->h);
    if (d == 0) return 4.0 * h2i;
    if (d == 1) return ((r % n) != n - 1) ? -h2i : 0.0;   /* (k+1, l) neighbour, same row l */
    if (d == n) return -h2i;                               /* (k, l+1) neighbour */
    return 0.0;
}

static void gram_factor(orc_ctx *c) {
    int n = c->n;
    long n2 = (long)n * n, bw = n + 1;
    for (long r = 0; r < n2; ++r)
        for (long d = 0; d <= n; ++d)
            c->U[r * bw + d] = (r + d < n2) ? gram_entry(c, r, d) : 0.0;
    /* Doolittle elimination: row i -= l_ik row k, l_ik = A(i,k)/A(k,k) = U(k,i)/U(k,k). */
    for (long k = 0; k < n2; ++k) {
        const double *uk = c->U + k * bw;
        long iend = k + n < n2 - 1 ? k + n : n2 - 1;
#pragma omp parallel for schedule(static) if (n >= 48)
        for (long i = k + 1; i <= iend; ++i) {
            double lik = uk[i - k] / uk[0];
            if (lik == 0.0) continue;
            double *ui = c->U + i * bw;
            long jend = k + n < n2 - 1 ? k + n : n2 - 1;
            for (long j = i; j <= jend; ++j) ui[j - i] -= lik * uk[j - k];
        }
    }
}

/* q = G^-1 rhs by forward (L z = rhs) and back (U q = z) substitution; n^2 arrays. */
void orc_gram_solve(const orc_ctx *c, const double *rhs, double *q) {
    int n = c->n;
    long n2 = (long)n * n, bw = n + 1;
    double *z = (double *)malloc(sizeof(double) * n2);
    for (long i = 0; i < n2; ++i) {
        double s = rhs[i];
        long k0 = i - n > 0 ? i - n : 0;
        for (long k = k0; k < i; ++k) {
            const double *uk = c->U + k * bw;
            s -= (uk[i - k] / uk[0]) * z[k];
        }
        z[i] = s;
    }
    for (long i = n2 - 1; i >= 0; --i) {
        const double *ui = c->U + i * bw;
        double s = z[i];
        long jend = i + n < n2 - 1 ? i + n : n2 - 1;
        for (long j = i + 1; j <= jend; ++j) s -= ui[j - i] * q[j];
        q[i] = s / ui[0];
    }
    free(z);
}

/* out = G v straight from Eq. 26 (test hook for P1). */
void orc_gram_matvec(const orc_ctx *c, const double *v, double *out) {
    int n = c->n;
    double h2i = 1.0 / (c->h * c->h);
    for (int l = 0; l < n; ++l)
        for (int k = 0; k < n; ++k) {
            long r = (long)l * n + k;
            double s = 4.0 * v[r];
            if (k > 0) s -= v[r - 1];
            if (k < n - 1) s -= v[r + 1];
            if (l > 0) s -= v[r - n];
            if (l < n - 1) s -= v[r + n];
            out[r] = h2i * s;
        }
}

/* ---------------------------------------------------------------- context */
orc_ctx *orc_create(int N, int nl, const int *widths, const float *K, const float *S,
                    const float *f, const float *theta0, double mobility, double lr,
                    double beta1, double beta2, double eps, int factor_gram, double gravity,
                    double rho_ratio) {
    if (N < 2 || nl < 1 || nl > ORC_MAX_LAYERS) return NULL;
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->N = N; c->n = N - 1; c->h = 1.0 / N; c->nl = nl;
    c->mobility = mobility; c->lr = lr; c->beta1 = beta1; c->beta2 = beta2; c->eps = eps;
    c->gravity = gravity; c->rho_ratio = rho_ratio;
    long np = 0;
    for (int l = 0; l <= nl; ++l) c->widths[l] = widths[l];
    for (int l = 0; l < nl; ++l) {
        c->woff[l] = np; np += (long)widths[l + 1] * widths[l];
        c->boff[l] = np; np += widths[l + 1];
    }
    c->np = np;
    long nn = (long)(N + 1) * (N + 1);
    c->alpha = (double *)malloc(sizeof(double) * nn);
    c->b = (double *)malloc(sizeof(double) * nn);
    c->f = (double *)malloc(sizeof(double) * nn);
    for (long p = 0; p < nn; ++p) c->f[p] = (double)f[p];
    set_alpha(c, K, S);
    set_rhs(c, K, S);
    c->theta = (double *)calloc(np, sizeof(double));
    c->m = (double *)calloc(np, sizeof(double));
    c->v = (double *)calloc(np, sizeof(double));
    if (theta0) for (long i = 0; i < np; ++i) c->theta[i] = (double)theta0[i];
    c->t = 0;
    if (factor_gram) {
        long n2 = (long)c->n * c->n;
        c->U = (double *)malloc(sizeof(double) * n2 * (c->n + 1));
        if (!c->U) { free(c->alpha); free(c->b); free(c->f); free(c->theta); free(c->m); free(c->v); free(c); return NULL; }
        gram_factor(c);
    }
    return c;
}

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    free(c->alpha); free(c->b); free(c->f); free(c->U); free(c->theta); free(c->m); free(c->v);
    free(c);
}

long orc_num_params(const orc_ctx *c) { return c->np; }
void orc_get_theta(const orc_ctx *c, double *th) { memcpy(th, c->theta, sizeof(double) * c->np); }
void orc_set_theta(orc_ctx *c, const double *th) { memcpy(c->theta, th, sizeof(double) * c->np); }
void orc_get_adam(const orc_ctx *c, double *m, double *v, long *t) {
    memcpy(m, c->m, sizeof(double) * c->np); memcpy(v, c->v, sizeof(double) * c->np); *t = c->t;
}
void orc_set_adam(orc_ctx *c, const double *m, const double *v, long t) {
    memcpy(c->m, m, sizeof(double) * c->np); memcpy(c->v, v, sizeof(double) * c->np); c->t = t;
}
void orc_get_alpha(const orc_ctx *c, double *a) {
    memcpy(a, c->alpha, sizeof(double) * (c->N + 1) * (c->N + 1));
}

/* ---------------------------------------------------------------- A1: network */
static int max_width(const orc_ctx *c) {
    int w = 0;
    for (int l = 0; l <= c->nl; ++l) if (c->widths[l] > w) w = c->widths[l];
    return w;
}

/* Forward pass at one point; act[l] receives the post-activation of layer l (act[0] = input).
 * Returns net (linear output layer). */
static double net_point(const orc_ctx *c, const double *th, double x, double y, double **act) {
    act[0][0] = x; act[0][1] = y;
    for (int l = 0; l < c->nl; ++l) {
        int fin = c->widths[l], fout = c->widths[l + 1];
        const double *W = th + c->woff[l], *bb = th + c->boff[l];
        for (int r = 0; r < fout; ++r) {
            double z = bb[r];
            for (int k = 0; k < fin; ++k) z += W[(long)r * fin + k] * act[l][k];
            act[l + 1][r] = (l + 1 < c->nl) ? tanh(z) : z;
        }
    }
    return act[c->nl][0];
}

static double cutoff(double x, double y) { return 16.0 * x * (1.0 - x) * y * (1.0 - y); }

static double **alloc_act(const orc_ctx *c) {
    int w = max_width(c);
    double **a = (double **)malloc(sizeof(double *) * (c->nl + 1));
    for (int l = 0; l <= c->nl; ++l) a[l] = (double *)malloc(sizeof(double) * w);
    return a;
}
static void free_act(const orc_ctx *c, double **a) {
    for (int l = 0; l <= c->nl; ++l) free(a[l]);
    free(a);
}

/* u at the interior nodes of rows j in [j0, j1) (clipped to [1, N-1]); every other node 0. One shard's
 * forward of the point-sharded iteration; pinned by P20 (additivity). */
void orc_forward_rows(const orc_ctx *c, const double *th, int j0, int j1, double *u) {
    int N = c->N;
    long nn = (long)(N + 1) * (N + 1);
    for (long p = 0; p < nn; ++p) u[p] = 0.0;
    if (j0 < 1) j0 = 1;
    if (j1 > N) j1 = N;
#pragma omp parallel
    {
        double **act = alloc_act(c);
#pragma omp for schedule(static)
        for (int j = j0; j < j1; ++j)
            for (int i = 1; i < N; ++i) {
                double x = (double)i / N, y = (double)j / N;
                u[idx(c, i, j)] = cutoff(x, y) * net_point(c, th, x, y, act);
            }
        free_act(c, act);
    }
}

/* u on the full (N+1)^2 lattice; boundary nodes are exactly 0 (cutoff). */
void orc_forward(const orc_ctx *c, const double *th, double *u) { orc_forward_rows(c, th, 1, c->N, u); }

/* Continuous evaluation at arbitrary points: out[p] = cutoff(x_p, y_p) net(x_p, y_p). */
void orc_eval_points(const orc_ctx *c, const double *th, long n, const double *xy, double *out) {
#pragma omp parallel
    {
        double **act = alloc_act(c);
#pragma omp for schedule(static)
        for (long p = 0; p < n; ++p) {
            double x = xy[2 * p], y = xy[2 * p + 1];
            out[p] = cutoff(x, y) * net_point(c, th, x, y, act);
        }
        free_act(c, act);
    }
}

/* ---------------------------------------------------------------- A2: residual (Eq. 25) */
/* res is n x n, res[(l-1) n + (k-1)] for interior test (k,l). */
void orc_residual(const orc_ctx *c, const double *u, double *res) {
    int N = c->N, n = c->n;
    double h = c->h, h2 = h * h;
    for (int l = 1; l < N; ++l)
        for (int k = 1; k < N; ++k) {
            /* the three nodes p where grad+ delta_kl != 0, with grad+ delta_kl(p): */
            const int pi[3] = {k, k - 1, k};
            const int pj[3] = {l, l, l - 1};
            const double dx[3] = {-1.0 / h, 1.0 / h, 0.0};
            const double dy[3] = {-1.0 / h, 0.0, 1.0 / h};
            double s = 0.0;
            for (int t = 0; t < 3; ++t) {
                int i = pi[t], j = pj[t];
                double gx = (u[idx(c, i + 1, j)] - u[idx(c, i, j)]) / h;   /* grad_x+ u (Eq. 22) */
                double gy = (u[idx(c, i, j + 1)] - u[idx(c, i, j)]) / h;   /* grad_y+ u */
                s += c->alpha[idx(c, i, j)] * (gx * dx[t] + gy * dy[t]);
            }
            /* (alpha grad+ u, grad+ delta)_h - (RHS, delta)_h, both with the h^2 weight */
            res[(long)(l - 1) * n + (k - 1)] = h2 * s - c->b[idx(c, k, l)];
        }
}

/* ---------------------------------------------------------------- A5: adjoint */
/* gu (full lattice) = sum_kl w_kl dRES_kl/du (transpose of orc_residual, scatter form). */
void orc_residual_adjoint(const orc_ctx *c, const double *w, double *gu) {
    int N = c->N, n = c->n;
    double h = c->h, h2 = h * h;
    long nn = (long)(N + 1) * (N + 1);
    for (long p = 0; p < nn; ++p) gu[p] = 0.0;
    for (int l = 1; l < N; ++l)
        for (int k = 1; k < N; ++k) {
            double wk = w[(long)(l - 1) * n + (k - 1)];
            const int pi[3] = {k, k - 1, k};
            const int pj[3] = {l, l, l - 1};
            const double dx[3] = {-1.0 / h, 1.0 / h, 0.0};
            const double dy[3] = {-1.0 / h, 0.0, 1.0 / h};
            for (int t = 0; t < 3; ++t) {
                int i = pi[t], j = pj[t];
                double a = h2 * c->alpha[idx(c, i, j)] * wk;
                /* d/du of a*(gx*dx + gy*dy) with gx = (u[i+1,j]-u[i,j])/h, gy = (u[i,j+1]-u[i,j])/h */
                gu[idx(c, i + 1, j)] += a * dx[t] / h;
                gu[idx(c, i, j)] -= a * dx[t] / h;
                gu[idx(c, i, j + 1)] += a * dy[t] / h;
                gu[idx(c, i, j)] -= a * dy[t] / h;
            }
        }
}

/* LOSS of a lattice function u (Eq. 27 via Eq. 28). Optional outputs res, q (n^2). */
double orc_loss_u(const orc_ctx *c, const double *u, double *res_out, double *q_out) {
    long n2 = (long)c->n * c->n;
    double *res = res_out ? res_out : (double *)malloc(sizeof(double) * n2);
    double *q = q_out ? q_out : (double *)malloc(sizeof(double) * n2);
    orc_residual(c, u, res);
    orc_gram_solve(c, res, q);
    double loss = 0.0;
    for (long i = 0; i < n2; ++i) loss += res[i] * q[i];
    if (!res_out) free(res);
    if (!q_out) free(q);
    return loss;
}

/* ---------------------------------------------------------------- A1-A6: loss and gradient */
/* dLOSS/dtheta summed over the MLP points of rows j in [j0, j1) (clipped to [1, N-1]), given
 * gu = dLOSS/du on the lattice: the chain rule through u = cutoff * net (A6, backpropagation).
 * One shard's backward; pinned by P20 (the shares sum to the gradient). */
void orc_grad_rows(const orc_ctx *c, const double *th, const double *gu, int j0, int j1, double *grad) {
    int N = c->N;
    if (j0 < 1) j0 = 1;
    if (j1 > N) j1 = N;
    int nthr = 1;
#ifdef _OPENMP
    nthr = omp_get_max_threads();
#endif
    long np = c->np;
    double *part = (double *)calloc((size_t)nthr * np, sizeof(double));
    int w = max_width(c);
#pragma omp parallel num_threads(nthr)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *g = part + (long)tid * np;
        double **act = alloc_act(c);
        double *dl = (double *)malloc(sizeof(double) * w);   /* delta of current layer */
        double *dp = (double *)malloc(sizeof(double) * w);   /* delta of previous layer */
#pragma omp for schedule(static)
        for (int j = j0; j < j1; ++j)
            for (int i = 1; i < N; ++i) {
                double x = (double)i / N, y = (double)j / N;
                net_point(c, th, x, y, act);
                /* u = cutoff * net  =>  dLOSS/dnet = gu * cutoff */
                dl[0] = gu[idx(c, i, j)] * cutoff(x, y);
                for (int l = c->nl - 1; l >= 0; --l) {
                    int fin = c->widths[l], fout = c->widths[l + 1];
                    const double *W = th + c->woff[l];
                    double *gW = g + c->woff[l], *gb = g + c->boff[l];
                    for (int r = 0; r < fout; ++r) {
                        gb[r] += dl[r];
                        for (int k = 0; k < fin; ++k) gW[(long)r * fin + k] += dl[r] * act[l][k];
                    }
                    if (l > 0) {
                        for (int k = 0; k < fin; ++k) {
                            double s = 0.0;
                            for (int r = 0; r < fout; ++r) s += W[(long)r * fin + k] * dl[r];
                            dp[k] = s * (1.0 - act[l][k] * act[l][k]);   /* tanh' */
                        }
                        double *tmp = dl; dl = dp; dp = tmp;
                    }
                }
            }
        free(dl); free(dp);
        free_act(c, act);
    }
    for (long k = 0; k < np; ++k) {
        double s = 0.0;
        for (int t = 0; t < nthr; ++t) s += part[(long)t * np + k];   /* thread order */
        grad[k] = s;
    }
    free(part);
}

double orc_loss_grad(const orc_ctx *c, const double *th_in, double *grad,
                     double *u_out, double *res_out, double *q_out, double *gu_out) {
    int N = c->N;
    long nn = (long)(N + 1) * (N + 1), n2 = (long)c->n * c->n;
    const double *th = th_in ? th_in : c->theta;
    double *u = u_out ? u_out : (double *)malloc(sizeof(double) * nn);
    double *res = res_out ? res_out : (double *)malloc(sizeof(double) * n2);
    double *q = q_out ? q_out : (double *)malloc(sizeof(double) * n2);
    double *gu = gu_out ? gu_out : (double *)malloc(sizeof(double) * nn);
    orc_forward(c, th, u);
    double loss = orc_loss_u(c, u, res, q);
    /* dLOSS/dRES = 2 G^-1 RES = 2 q (G symmetric) */
    double *w2 = (double *)malloc(sizeof(double) * n2);
    for (long i = 0; i < n2; ++i) w2[i] = 2.0 * q[i];
    orc_residual_adjoint(c, w2, gu);
    free(w2);
    if (grad) orc_grad_rows(c, th, gu, 1, N, grad);
    if (!u_out) free(u);
    if (!res_out) free(res);
    if (!q_out) free(q);
    if (!gu_out) free(gu);
    return loss;
}

/* ---------------------------------------------------------------- A8: Adam */
void orc_adam_step(orc_ctx *c, const double *g) {
    c->t += 1;
    double bc1 = 1.0 - pow(c->beta1, (double)c->t);
    double bc2 = 1.0 - pow(c->beta2, (double)c->t);
    for (long k = 0; k < c->np; ++k) {
        c->m[k] = c->beta1 * c->m[k] + (1.0 - c->beta1) * g[k];
        c->v[k] = c->beta2 * c->v[k] + (1.0 - c->beta2) * g[k] * g[k];
        double mh = c->m[k] / bc1, vh = c->v[k] / bc2;
        c->theta[k] -= c->lr * mh / (sqrt(vh) + c->eps);
    }
}

/* n Adam iterations; hist[k] = LOSS before the (k+1)-th update. */
int orc_train(orc_ctx *c, int n_iters, double *hist) {
    double *g = (double *)malloc(sizeof(double) * c->np);
    for (int k = 0; k < n_iters; ++k) {
        double loss = orc_loss_grad(c, NULL, g, NULL, NULL, NULL, NULL);
        if (hist) hist[k] = loss;
        if (!isfinite(loss)) { free(g); return -4; }
        orc_adam_step(c, g);
    }
    free(g);
    return 0;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
