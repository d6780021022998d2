/*
 * iga_oracle.c -- plain, slow, fp64 CPU ORACLE of the IGA-ADS saturation step.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as crvpinn_oracle.c): only tests/, __graft_entry__ and
 * bench.py's oracle legs may load it; it shares nothing with the CUDA path.
 *
 * What it computes, in the paper's order (§3-§4):
 *   space   tensor-product B-splines of degree r, C^{r-1}, open uniform knots on [0,1] with Ne
 *           elements per axis, nb = Ne + r functions per axis (Eq. 11);
 *           basis values/derivatives by the Cox-de Boor recursion (textbook); Gauss-Legendre
 *           quadrature with r+1 points per element and axis (reading R27; exact for the mass matrix).
 *   mass    M = M^x (x) M^y, M^x_ik = int B_i B_k dx (Eq. 14); here M^x = M^y,
 *           a DENSE matrix solved by Gaussian elimination with partial pivoting (no banded trick:
 *           the oracle does not rely on the "Thomas algorithm" claim).
 *   project (C, B_kl) = (f, B_kl) for every (k,l): C = M^-1 L, L_kl = sum over elements and Gauss
 *           points of w f B_k B_l (the isogeometric L2 projection of Eq. 12-13).
 *   step    Eq. 10 non-dimensionalised like the pressure (readings R24, R25):
 *           (S^{n+1}, v) = (S^n, v) + (tau/phi) ( -M S^n K (grad p . grad v + r Gr v_y) + q v ),
 *           M = mu_w/mu_g, r = rho_g/rho_w, Gr the gravity number of R23, K and q constant per
 *           element, phi a scalar; the boundary coefficients of S^{n+1} are set to 0 after the solve
 *           (zero Dirichlet saturation; reading R26).
 *   eval    field value and gradient at arbitrary points (Eq. 16).
 * Pins: tests/test_oracle_pins.py P17-P19.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct iga_ctx {
    int ne, r, nb;
    double *knots;      /* ne + 2r + 1 */
    double *gx, *gw;    /* Gauss points/weights on [0,1], r+1 */
    double *M;          /* dense nb x nb mass matrix (1D) */
} iga_ctx;

/* Gauss-Legendre on [0,1] with m points: Newton on P_m from the Chebyshev guess. */
static void gauss_legendre(int m, double *x, double *w) {
    for (int i = 0; i < m; ++i) {
        double z = cos(M_PI * (i + 0.75) / (m + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;
            for (int k = 2; k <= m; ++k) {
                double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            if (m == 1) { p1 = z; p0 = 1.0; }
            dp = m * (z * p1 - p0) / (z * z - 1.0);
            double dz = p1 / dp;
            z -= dz;
            if (fabs(dz) < 1e-16) break;
        }
        x[m - 1 - i] = 0.5 * (1.0 + z);
        w[m - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);   /* 2/((1-z^2) P'^2) on [-1,1], halved */
    }
}

/* Cox-de Boor: the r+1 non-zero basis functions at x and their first derivatives.
 * Returns the index of the first one (span - r). */
static int basis_at(const iga_ctx *c, double x, double *val, double *der) {
    int r = c->r, ne = c->ne;
    int e = (int)floor(x * ne);
    if (e < 0) e = 0;
    if (e > ne - 1) e = ne - 1;
    int span = e + r;   /* knots[span] <= x < knots[span+1] */
    const double *U = c->knots;
    double N[16][16];   /* N[p][j]: degree-p functions, local index j */
    N[0][0] = 1.0;
    for (int p = 1; p <= r; ++p) {
        for (int j = 0; j <= p; ++j) {
            double v = 0.0;
            int i = span - p + j;   /* global index of function j of degree p */
            if (j >= 1) {           /* term with N_{i,p-1} */
                double d = U[i + p] - U[i];
                if (d > 0.0) v += (x - U[i]) / d * N[p - 1][j - 1];
            }
            if (j <= p - 1) {       /* term with N_{i+1,p-1} */
                double d = U[i + p + 1] - U[i + 1];
                if (d > 0.0) v += (U[i + p + 1] - x) / d * N[p - 1][j];
            }
            N[p][j] = v;
        }
    }
    for (int j = 0; j <= r; ++j) {
        val[j] = N[r][j];
        int i = span - r + j;
        double d = 0.0;
        if (j >= 1) {
            double den = U[i + r] - U[i];
            if (den > 0.0) d += r / den * N[r - 1][j - 1];
        }
        if (j <= r - 1) {
            double den = U[i + r + 1] - U[i + 1];
            if (den > 0.0) d -= r / den * N[r - 1][j];
        }
        der[j] = d;
    }
    return span - r;
}

iga_ctx *iga_create(int ne, int r) {
    if (ne < 1 || r < 1 || r > 8) return NULL;
    iga_ctx *c = (iga_ctx *)calloc(1, sizeof(iga_ctx));
    c->ne = ne; c->r = r; c->nb = ne + r;
    int nk = ne + 2 * r + 1;
    c->knots = (double *)malloc(sizeof(double) * nk);
    for (int i = 0; i < nk; ++i) {
        int k = i - r;
        if (k < 0) k = 0;
        if (k > ne) k = ne;
        c->knots[i] = (double)k / ne;
    }
    c->gx = (double *)malloc(sizeof(double) * (r + 1));
    c->gw = (double *)malloc(sizeof(double) * (r + 1));
    gauss_legendre(r + 1, c->gx, c->gw);
    int nb = c->nb;
    c->M = (double *)calloc((size_t)nb * nb, sizeof(double));
    double val[16], der[16];
    for (int e = 0; e < ne; ++e)
        for (int q = 0; q <= r; ++q) {
            double x = (e + c->gx[q]) / ne, w = c->gw[q] / ne;
            int i0 = basis_at(c, x, val, der);
            for (int a = 0; a <= r; ++a)
                for (int b = 0; b <= r; ++b) c->M[(size_t)(i0 + a) * nb + (i0 + b)] += w * val[a] * val[b];
        }
    return c;
}

void iga_destroy(iga_ctx *c) {
    if (!c) return;
    free(c->knots); free(c->gx); free(c->gw); free(c->M);
    free(c);
}

int iga_num_basis(const iga_ctx *c) { return c->nb; }
void iga_mass_1d(const iga_ctx *c, double *out) { memcpy(out, c->M, sizeof(double) * c->nb * c->nb); }
void iga_gauss(const iga_ctx *c, double *x, double *w) {
    memcpy(x, c->gx, sizeof(double) * (c->r + 1));
    memcpy(w, c->gw, sizeof(double) * (c->r + 1));
}
int iga_basis(const iga_ctx *c, double x, double *val, double *der) { return basis_at(c, x, val, der); }

/* Quadrature points of the tensor rule, x fastest: index ((ey(r+1)+qy) ne(r+1)) + ex(r+1) + qx. */
void iga_quad_points(const iga_ctx *c, double *xy) {
    int r = c->r, ne = c->ne, m = ne * (r + 1);
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
            long p = (long)j * m + i;
            xy[2 * p] = (i / (r + 1) + c->gx[i % (r + 1)]) / ne;
            xy[2 * p + 1] = (j / (r + 1) + c->gx[j % (r + 1)]) / ne;
        }
}

/* X = M^-1 B for nrhs right-hand sides (columns of B, B is nb x nrhs row-major), dense GE with
 * partial pivoting on a copy of M. */
static void dense_solve(const iga_ctx *c, double *B, int nrhs) {
    int n = c->nb;
    double *A = (double *)malloc(sizeof(double) * n * n);
    memcpy(A, c->M, sizeof(double) * n * n);
    for (int k = 0; k < n; ++k) {
        int piv = k;
        for (int i = k + 1; i < n; ++i)
            if (fabs(A[(size_t)i * n + k]) > fabs(A[(size_t)piv * n + k])) piv = i;
        if (piv != k) {
            for (int j = 0; j < n; ++j) { double t = A[(size_t)k * n + j]; A[(size_t)k * n + j] = A[(size_t)piv * n + j]; A[(size_t)piv * n + j] = t; }
            for (int j = 0; j < nrhs; ++j) { double t = B[(size_t)k * nrhs + j]; B[(size_t)k * nrhs + j] = B[(size_t)piv * nrhs + j]; B[(size_t)piv * nrhs + j] = t; }
        }
        for (int i = k + 1; i < n; ++i) {
            double l = A[(size_t)i * n + k] / A[(size_t)k * n + k];
            if (l == 0.0) continue;
            for (int j = k; j < n; ++j) A[(size_t)i * n + j] -= l * A[(size_t)k * n + j];
            for (int j = 0; j < nrhs; ++j) B[(size_t)i * nrhs + j] -= l * B[(size_t)k * nrhs + j];
        }
    }
    for (int k = n - 1; k >= 0; --k)
        for (int j = 0; j < nrhs; ++j) {
            double s = B[(size_t)k * nrhs + j];
            for (int i = k + 1; i < n; ++i) s -= A[(size_t)k * n + i] * B[(size_t)i * nrhs + j];
            B[(size_t)k * nrhs + j] = s / A[(size_t)k * n + k];
        }
    free(A);
}

/* C = (M^x (x) M^y)^-1 L with L, C stored [l][k] (row = y index, column = x index):
 * C = M^-1 L M^-T (M symmetric): solve along y (columns of the [l][k] matrix), then along x. */
void iga_kron_solve(const iga_ctx *c, const double *L, double *C) {
    int n = c->nb;
    double *T = (double *)malloc(sizeof(double) * n * n);
    memcpy(T, L, sizeof(double) * n * n);
    dense_solve(c, T, n);                  /* T = M^-1 L (acts on the row index l) */
    for (int l = 0; l < n; ++l)            /* transpose */
        for (int k = 0; k < n; ++k) C[(size_t)k * n + l] = T[(size_t)l * n + k];
    dense_solve(c, C, n);                  /* acts on the x index */
    for (int l = 0; l < n; ++l)
        for (int k = l + 1; k < n; ++k) { double t = C[(size_t)l * n + k]; C[(size_t)l * n + k] = C[(size_t)k * n + l]; C[(size_t)k * n + l] = t; }
    free(T);
}

/* Load L[l][k] = int f B_k(x) B_l(y) by the tensor Gauss rule; f at the quadrature points. */
void iga_load(const iga_ctx *c, const double *fq, double *L) {
    int r = c->r, ne = c->ne, n = c->nb, m = ne * (r + 1);
    double vx[16], dx[16], vy[16], dy[16];
    memset(L, 0, sizeof(double) * n * n);
    for (int j = 0; j < m; ++j) {
        double y = (j / (r + 1) + c->gx[j % (r + 1)]) / ne, wy = c->gw[j % (r + 1)] / ne;
        int l0 = basis_at(c, y, vy, dy);
        for (int i = 0; i < m; ++i) {
            double x = (i / (r + 1) + c->gx[i % (r + 1)]) / ne, wx = c->gw[i % (r + 1)] / ne;
            int k0 = basis_at(c, x, vx, dx);
            double f = fq[(long)j * m + i] * wx * wy;
            for (int b = 0; b <= r; ++b)
                for (int a = 0; a <= r; ++a) L[(size_t)(l0 + b) * n + (k0 + a)] += f * vx[a] * vy[b];
        }
    }
}

void iga_project(const iga_ctx *c, const double *fq, double *C) {
    int n = c->nb;
    double *L = (double *)malloc(sizeof(double) * n * n);
    iga_load(c, fq, L);
    iga_kron_solve(c, L, C);
    free(L);
}

/* value (and gradient if grad != NULL) of the field with coefficients C[l][k] at (x, y) */
void iga_eval(const iga_ctx *c, const double *C, long npts, const double *xy, double *val, double *grad) {
    int r = c->r, n = c->nb;
    double vx[16], dx[16], vy[16], dy[16];
    for (long p = 0; p < npts; ++p) {
        int k0 = basis_at(c, xy[2 * p], vx, dx), l0 = basis_at(c, xy[2 * p + 1], vy, dy);
        double v = 0.0, gx = 0.0, gy = 0.0;
        for (int b = 0; b <= r; ++b)
            for (int a = 0; a <= r; ++a) {
                double cc = C[(size_t)(l0 + b) * n + (k0 + a)];
                v += cc * vx[a] * vy[b];
                gx += cc * dx[a] * vy[b];
                gy += cc * vx[a] * dy[b];
            }
        val[p] = v;
        if (grad) { grad[2 * p] = gx; grad[2 * p + 1] = gy; }
    }
}

/* One explicit saturation step (Eq. 10 with readings R24-R26). S, P, S_out: coefficients [l][k];
 * K, q: per element [ey][ex]. */
void iga_saturation_step(const iga_ctx *c, const double *S, const double *P, const double *K, const double *q,
                         double tau, double phi, double mobility, double rho_ratio, double gravity, double *S_out) {
    int r = c->r, ne = c->ne, n = c->nb, m = ne * (r + 1);
    double vx[16], dx[16], vy[16], dy[16];
    double *L = (double *)calloc((size_t)n * n, sizeof(double));
    for (int j = 0; j < m; ++j) {
        int ey = j / (r + 1);
        double y = (ey + c->gx[j % (r + 1)]) / ne, wy = c->gw[j % (r + 1)] / ne;
        int l0 = basis_at(c, y, vy, dy);
        for (int i = 0; i < m; ++i) {
            int ex = i / (r + 1);
            double x = (ex + c->gx[i % (r + 1)]) / ne, wx = c->gw[i % (r + 1)] / ne;
            int k0 = basis_at(c, x, vx, dx);
            double s = 0.0, px = 0.0, py = 0.0;
            for (int b = 0; b <= r; ++b)
                for (int a = 0; a <= r; ++a) {
                    s += S[(size_t)(l0 + b) * n + (k0 + a)] * vx[a] * vy[b];
                    px += P[(size_t)(l0 + b) * n + (k0 + a)] * dx[a] * vy[b];
                    py += P[(size_t)(l0 + b) * n + (k0 + a)] * vx[a] * dy[b];
                }
            double Ke = K[(size_t)ey * ne + ex], qe = q[(size_t)ey * ne + ex], w = wx * wy;
            double mob = mobility * s * Ke;
            /* integrand, tested with v = B_k(x) B_l(y): S v + (tau/phi)(-mob (p_x v_x + (p_y + r Gr) v_y) + q v) */
            for (int b = 0; b <= r; ++b)
                for (int a = 0; a <= r; ++a) {
                    double v = vx[a] * vy[b], v_x = dx[a] * vy[b], v_y = vx[a] * dy[b];
                    double f = s * v + tau / phi * (-mob * (px * v_x + (py + rho_ratio * gravity) * v_y) + qe * v);
                    L[(size_t)(l0 + b) * n + (k0 + a)] += w * f;
                }
        }
    }
    iga_kron_solve(c, L, S_out);
    for (int k = 0; k < n; ++k) {
        S_out[k] = 0.0;
        S_out[(size_t)(n - 1) * n + k] = 0.0;
        S_out[(size_t)k * n] = 0.0;
        S_out[(size_t)k * n + n - 1] = 0.0;
    }
    free(L);
}
