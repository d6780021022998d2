// iga.cu -- SURVEY.md §8(f) f3: the IGA-ADS explicit saturation step on the GPU (§3-§4).
//
// Tensor-product B-splines of degree r (C^{r-1}, open uniform knots, ne elements per axis,
// nb = ne + r functions per axis; Eq. 11), Gauss-Legendre with r+1 points per element and axis
// (reading R27). One step of Eq. 10 (readings R24-R26):
//   (S^{n+1}, v) = (S^n, v) + (tau/phi) ( -M S^n K (grad p . grad v + r Gr v_y) + q v )   for all v,
//   M = M^x (x) M^y (Eq. 14)  =>  S^{n+1} = M^-1 (load), solved direction by direction,
// then the boundary coefficients are set to 0 (zero Dirichlet saturation).
// Kernels:
//   k_iga_qp      one thread per quadrature point: S^n, grad p^n from the local (r+1)^2 coefficient
//                 stencil; the integrand's weights for v, v_x, v_y (or f w for a plain projection)
//   k_iga_gather  one thread per test function (k,l): sums its (r+1)^2 elements x (r+1)^2 points in a
//                 fixed order (deterministic, no atomics) -> the load matrix L[l][k]
//   k_iga_band    one thread per column (fp64): (LDL^T)^-1 along the row index with the precomputed band
//                 factors of the 1D mass matrix (bandwidth r; the paper's "Thomas algorithm",
//                 PAPER.md:209, generalised to bandwidth r); coalesced across threads
//   k_iga_transpose, k_iga_dirichlet, k_iga_eval (field value/gradient at arbitrary points)
// Coefficient matrices are [l][k] (row = y basis index). Host buffers at the C ABI.
#include "common.cuh"
#include "../../include/crvpinn.h"
#include <cstdlib>
#include <type_traits>
#include <cstring>
#include <cmath>
#include <string>
#include <vector>

namespace crv {
namespace {

constexpr int IGA_MAX_R = 6;

struct IgaDev {
    int ne = 0, r = 0, nb = 0, m = 0;   // m = ne (r+1) quadrature points per axis
    float *bv = nullptr, *bd = nullptr; // [ne][r+1 points][r+1 functions] values / x-derivatives
    float *gw = nullptr;                // [m] weights (x quadrature incl. 1/ne), same for y
    double *lf = nullptr;               // [nb][r] sub-diagonal band of the unit lower factor (row i: L_{i,i-1..i-r})
    double *dinv = nullptr;             // [nb] 1/D of LDL^T
    int nseg = 0;                       // k_iga_band_seg: segments per column (0: not used)
    int *seg0 = nullptr;                // [nseg + 1] segment starts
    double *cfw = nullptr, *cbw = nullptr;   // [nb][r] homogeneous responses of the forward / backward
                                             // substitution to the state at the segment's entry
    float *qv = nullptr;                // [3][m*m] integrand weights
    double *A = nullptr, *B = nullptr;  // nb*nb work matrices: the mass solves run in fp64 (the degree-3
                                        // mass matrix loses ~4 digits to conditioning in fp32)
    float *outf = nullptr;              // nb*nb fp32 result
    float *io = nullptr;                // staging for inputs/outputs (grown on demand)
    size_t io_cap = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    float last_ms = 0.f;
};

// ---------------------------------------------------------------- host precomputation
// Gauss-Legendre nodes/weights on [0,1]: Newton on the three-term recurrence of P_m.
void gauss01(int m, std::vector<double> &x, std::vector<double> &w) {
    x.assign(m, 0.0);
    w.assign(m, 0.0);
    for (int i = 0; i < m; ++i) {
        double t = std::cos(M_PI * (4.0 * i + 3.0) / (4.0 * m + 2.0));
        double dp = 1.0;
        for (int it = 0; it < 64; ++it) {
            double pm1 = 1.0, p = t;   // P_0, P_1
            for (int n = 1; n < m; ++n) {
                const double pn1 = ((2.0 * n + 1.0) * t * p - n * pm1) / (n + 1.0);
                pm1 = p;
                p = pn1;
            }
            dp = m * (pm1 - t * p) / (1.0 - t * t);   // P_m'
            const double step = p / dp;
            t -= step;
            if (std::fabs(step) < 1e-16) break;
        }
        x[m - 1 - i] = 0.5 * (t + 1.0);
        w[m - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

// The r+1 non-zero B-splines of degree r at x (uniform open knots, ne elements) and their
// derivatives, by the triangular de Boor table (left/right differences); returns the first index.
int bspline_local(int ne, int r, double x, double *val, double *der) {
    auto knot = [&](int i) { return (double)std::min(std::max(i - r, 0), ne) / ne; };
    int e = (int)std::floor(x * ne);
    e = std::min(std::max(e, 0), ne - 1);
    const int span = e + r;
    std::vector<double> left(r + 1), right(r + 1);
    std::vector<std::vector<double>> nd(r + 1, std::vector<double>(r + 1, 0.0));
    nd[0][0] = 1.0;
    for (int j = 1; j <= r; ++j) {
        left[j] = x - knot(span + 1 - j);
        right[j] = knot(span + j) - x;
        double saved = 0.0;
        for (int s = 0; s < j; ++s) {
            const double den = right[s + 1] + left[j - s];
            const double tmp = den != 0.0 ? nd[j - 1][s] / den : 0.0;
            nd[j][s] = saved + right[s + 1] * tmp;
            saved = left[j - s] * tmp;
        }
        nd[j][j] = saved;
    }
    for (int a = 0; a <= r; ++a) val[a] = nd[r][a];
    // derivative: r (N_{i,r-1}/(u_{i+r}-u_i) - N_{i+1,r-1}/(u_{i+r+1}-u_{i+1}))
    for (int a = 0; a <= r; ++a) {
        const int i = span - r + a;
        double d = 0.0;
        if (a >= 1) {
            const double den = knot(i + r) - knot(i);
            if (den > 0.0) d += r * nd[r - 1][a - 1] / den;
        }
        if (a <= r - 1) {
            const double den = knot(i + r + 1) - knot(i + 1);
            if (den > 0.0) d -= r * nd[r - 1][a] / den;
        }
        der[a] = d;
    }
    return span - r;
}

// ---------------------------------------------------------------- kernels
// mode 0: saturation integrand; mode 1: plain projection (f given at the points)
__global__ void k_iga_qp(IgaDev g, const float *__restrict__ S, const float *__restrict__ P,
                         const float *__restrict__ K, const float *__restrict__ q, const float *__restrict__ fq,
                         int mode, float tau_phi, float mob, float grav_y) {
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long mm = (long)g.m * g.m;
    if (p >= mm) return;
    const int R1 = g.r + 1;
    const int j = (int)(p / g.m), i = (int)(p % g.m);
    const int ex = i / R1, qx = i % R1, ey = j / R1, qy = j % R1;
    const float w = g.gw[i] * g.gw[j];
    if (mode == 1) {
        g.qv[p] = w * fq[p];
        g.qv[mm + p] = 0.f;
        g.qv[2 * mm + p] = 0.f;
        return;
    }
    const float *bvx = g.bv + ((long)ex * R1 + qx) * R1, *bdx = g.bd + ((long)ex * R1 + qx) * R1;
    const float *bvy = g.bv + ((long)ey * R1 + qy) * R1, *bdy = g.bd + ((long)ey * R1 + qy) * R1;
    float s = 0.f, px = 0.f, py = 0.f;
    for (int b = 0; b < R1; ++b) {
        const float *srow = S + (long)(ey + b) * g.nb + ex, *prow = P + (long)(ey + b) * g.nb + ex;
        float ss = 0.f, ppx = 0.f, ppy = 0.f;
        for (int a = 0; a < R1; ++a) {
            ss = fmaf(srow[a], bvx[a], ss);
            ppx = fmaf(prow[a], bdx[a], ppx);
            ppy = fmaf(prow[a], bvx[a], ppy);
        }
        s = fmaf(ss, bvy[b], s);
        px = fmaf(ppx, bvy[b], px);
        py = fmaf(ppy, bdy[b], py);
    }
    const long e = (long)ey * g.ne + ex;
    const float flux = -tau_phi * mob * s * K[e];
    g.qv[p] = w * (s + tau_phi * q[e]);
    g.qv[mm + p] = w * flux * px;
    g.qv[2 * mm + p] = w * flux * (py + grav_y);
}

__global__ void k_iga_gather(IgaDev g, double *__restrict__ L) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)g.nb * g.nb) return;
    const int l = (int)(t / g.nb), k = (int)(t % g.nb);
    const int R1 = g.r + 1;
    const long mm = (long)g.m * g.m;
    double acc = 0.0;
    for (int ey = max(l - g.r, 0); ey <= min(l, g.ne - 1); ++ey) {
        const int b = l - ey;
        for (int qy = 0; qy < R1; ++qy) {
            const float vy = g.bv[((long)ey * R1 + qy) * R1 + b], dy = g.bd[((long)ey * R1 + qy) * R1 + b];
            const long row = (long)(ey * R1 + qy) * g.m;
            for (int ex = max(k - g.r, 0); ex <= min(k, g.ne - 1); ++ex) {
                const int a = k - ex;
                for (int qx = 0; qx < R1; ++qx) {
                    const float vx = g.bv[((long)ex * R1 + qx) * R1 + a], dx = g.bd[((long)ex * R1 + qx) * R1 + a];
                    const long p = row + ex * R1 + qx;
                    acc += (double)g.qv[p] * (double)(vx * vy) + (double)g.qv[mm + p] * (double)(dx * vy) +
                           (double)g.qv[2 * mm + p] * (double)(vx * dy);
                }
            }
        }
    }
    L[t] = acc;
}

// Fused integrand + load assembly (replaces k_iga_qp + k_iga_gather): a block owns TB x TB test
// functions (k, l), computes the integrand of k_iga_qp at every Gauss point of the elements their
// supports touch (a halo of r elements) into shared memory, and then each thread sums its test
// function's load, factorised by Gauss rows (fp32 row sums of at most (r+1)^2 terms, fp64 across
// rows). The 3 x m^2 integrand array never goes through HBM.
template <int TB, int RD>   // RD: the spline degree r (compile time: the per-point loops unroll)
__global__ void __launch_bounds__(TB * TB) k_iga_assemble(IgaDev g, const float *__restrict__ S,
                                                          const float *__restrict__ P, const float *__restrict__ K,
                                                          const float *__restrict__ q, const float *__restrict__ fq,
                                                          int mode, float tau_phi, float mob, float grav_y,
                                                          double *__restrict__ L) {
    extern __shared__ float sq[];   // [3][QW][QW] integrand of the block's Gauss points, then the staged inputs
    constexpr int r = RD, R1 = RD + 1, RR = R1 * R1, QW = (TB + r) * R1;
    const int ne = g.ne, nb = g.nb, m = g.m;
    const int k0 = blockIdx.x * TB, l0 = blockIdx.y * TB;
    const int ex0 = max(k0 - r, 0), ey0 = max(l0 - r, 0);                          // first element
    const int ex1 = min(k0 + TB - 1, ne - 1), ey1 = min(l0 + TB - 1, ne - 1);      // last element
    const int EX = ex1 - ex0 + 1, EY = ey1 - ey0 + 1;
    const int QX = EX * R1, QY = EY * R1;
    // staged inputs (one batched pass over global memory; every later read is shared memory):
    // basis values / x-derivatives of the x and y elements, Gauss weights, and (mode 0) the S and P
    // coefficient tiles and the element fields K, q; (mode 1) the values fq at the block's Gauss points
    float *sbx = sq + 3 * QW * QW, *sdx = sbx + EX * RR, *sby = sdx + EX * RR, *sdy = sby + EY * RR;
    float *sgx = sdy + EY * RR, *sgy = sgx + QX;
    const int CX = EX + r, CY = EY + r;
    float *sS = sgy + QY, *sP = sS + CX * CY, *sK = sP + CX * CY, *sQ = sK + EX * EY;
    float *sF = sS;   // mode 1: [QY][QX] in place of the mode-0 arrays
    {
        const int n1 = EX * RR, n2 = n1 + EX * RR, n3 = n2 + EY * RR, n4 = n3 + EY * RR, n5 = n4 + QX, n6 = n5 + QY;
        const int n7 = n6 + (mode == 1 ? 0 : CX * CY), n8 = n7 + (mode == 1 ? 0 : CX * CY);
        const int n9 = n8 + (mode == 1 ? 0 : EX * EY), n10 = n9 + (mode == 1 ? QX * QY : EX * EY);
        auto src = [&](int e) -> float {
            if (mode == 1 && e >= n6) {
                const int t = e - n6;
                return fq[(long)(ey0 * R1 + t / QX) * m + ex0 * R1 + t % QX];
            }
            if (e < n1) return g.bv[(long)ex0 * RR + e];
            if (e < n2) return g.bd[(long)ex0 * RR + (e - n1)];
            if (e < n3) return g.bv[(long)ey0 * RR + (e - n2)];
            if (e < n4) return g.bd[(long)ey0 * RR + (e - n3)];
            if (e < n5) return g.gw[ex0 * R1 + (e - n4)];
            if (e < n6) return g.gw[ey0 * R1 + (e - n5)];
            if (e < n8) {
                const int t = e < n7 ? e - n6 : e - n7;
                const int cy = t / CX, cx = t % CX;
                const int gy = min(ey0 + cy, nb - 1), gx = min(ex0 + cx, nb - 1);
                return (e < n7 ? S : P)[(long)gy * nb + gx];
            }
            const int t = e < n9 ? e - n8 : e - n9;
            const long el = (long)(ey0 + t / EX) * ne + ex0 + t % EX;
            return e < n9 ? K[el] : q[el];
        };
        const int step = (int)blockDim.x;
        for (int e0 = threadIdx.x; e0 < n10; e0 += 4 * step) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = e0 + u * step < n10 ? src(e0 + u * step) : 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (e0 + u * step < n10) sbx[e0 + u * step] = v[u];   // the staged arrays are contiguous
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < QX * QY; t += blockDim.x) {
        const int jy = t / QX, ix = t % QX;
        const int lex = ix / R1, qx = ix % R1, ley = jy / R1, qy = jy % R1;
        const float w = sgx[ix] * sgy[jy];
        float v0, v1, v2;
        if (mode == 1) {
            v0 = w * sF[jy * QX + ix];
            v1 = v2 = 0.f;
        } else {
            const float *bvx = sbx + (lex * R1 + qx) * R1, *bdx = sdx + (lex * R1 + qx) * R1;
            const float *bvy = sby + (ley * R1 + qy) * R1, *bdy = sdy + (ley * R1 + qy) * R1;
            float sv = 0.f, px = 0.f, py = 0.f;
#pragma unroll
            for (int b = 0; b < R1; ++b) {
                const float *srow = sS + (ley + b) * CX + lex, *prow = sP + (ley + b) * CX + lex;
                float ss = 0.f, ppx = 0.f, ppy = 0.f;
#pragma unroll
                for (int a = 0; a < R1; ++a) {
                    ss = fmaf(srow[a], bvx[a], ss);
                    ppx = fmaf(prow[a], bdx[a], ppx);
                    ppy = fmaf(prow[a], bvx[a], ppy);
                }
                sv = fmaf(ss, bvy[b], sv);
                px = fmaf(ppx, bvy[b], px);
                py = fmaf(ppy, bdy[b], py);
            }
            const int el = ley * EX + lex;
            const float flux = -tau_phi * mob * sv * sK[el];
            v0 = w * (sv + tau_phi * sQ[el]);
            v1 = w * flux * px;
            v2 = w * flux * (py + grav_y);
        }
        const int o = jy * QW + ix;
        sq[o] = v0;
        sq[QW * QW + o] = v1;
        sq[2 * QW * QW + o] = v2;
    }
    __syncthreads();
    const int k = k0 + (int)(threadIdx.x % TB), l = l0 + (int)(threadIdx.x / TB);
    if (k >= nb || l >= nb) return;
    // the x-direction test-function factors of this k in registers: element ex = exa + de of its
    // support (exa = max(k - r, 0)), Gauss point qx; zero where the support leaves the mesh
    const int exa = max(k - r, 0), nex = min(k, ne - 1) - exa + 1;
    float vxs[R1][R1], dxs[R1][R1];
#pragma unroll
    for (int de = 0; de < R1; ++de)
#pragma unroll
        for (int qx = 0; qx < R1; ++qx) {
            const bool ok = de < nex;
            const int o = ((ok ? exa + de - ex0 : 0) * R1 + qx) * R1 + (ok ? k - exa - de : 0);
            vxs[de][qx] = ok ? sbx[o] : 0.f;
            dxs[de][qx] = ok ? sdx[o] : 0.f;
        }
    // per Gauss row: A = sum_x (q0 vx + q1 dx), B = sum_x q2 vx in fp32 (at most (r+1)^2 terms),
    // then L += vy A + dy B in fp64 (two conversions per row instead of six per point)
    double acc = 0.0;
    const int xo = (exa - ex0) * R1;
    const int eya = max(l - r, 0), ney = min(l, ne - 1) - eya + 1;
#pragma unroll
    for (int de = 0; de < R1; ++de) {
        if (de >= ney) break;
        const int ey = eya + de, b = l - ey;
#pragma unroll
        for (int qy = 0; qy < R1; ++qy) {
            const float vy = sby[((ey - ey0) * R1 + qy) * R1 + b], dy = sdy[((ey - ey0) * R1 + qy) * R1 + b];
            const float *r0 = sq + ((ey - ey0) * R1 + qy) * QW + xo;
            // degree >= 4: the row sums in fp64 too (the mass matrix's condition number, ~5e3 in 2-D at
            // degree 4 and 2e5 at 6, amplifies the rounding of (r+1)^2-term fp32 sums visibly)
            using acc_t = typename std::conditional<(RD >= 4), double, float>::type;
            acc_t A = 0, B = 0;
#pragma unroll
            for (int dx2 = 0; dx2 < R1; ++dx2)
#pragma unroll
                for (int qx = 0; qx < R1; ++qx) {
                    const int t = (dx2 < nex ? dx2 : 0) * R1 + qx;   // zero factors beyond the mesh
                    A = fma((acc_t)r0[t], (acc_t)vxs[dx2][qx], A);
                    A = fma((acc_t)r0[QW * QW + t], (acc_t)dxs[dx2][qx], A);
                    B = fma((acc_t)r0[2 * QW * QW + t], (acc_t)vxs[dx2][qx], B);
                }
            acc = fma((double)vy, (double)A, acc);
            acc = fma((double)dy, (double)B, acc);
        }
    }
    L[(long)l * nb + k] = acc;
}

static bool assemble_split() {   // tuning knob: CRVPINN_IGA_ASSEMBLY=split -> k_iga_qp + k_iga_gather
    const char *e = getenv("CRVPINN_IGA_ASSEMBLY");
    return e && strcmp(e, "split") == 0;
}

template <int TB, int RD>
static void assemble_launch(IgaDev &g, const float *S, const float *P, const float *K, const float *q, const float *fq,
                            int mode, float tau_phi, float mob, float grav_y, cudaStream_t s) {
    constexpr int R1 = RD + 1, QW = (TB + RD) * R1, E = TB + RD, RR = R1 * R1;
    constexpr size_t smem = sizeof(float) * (3 * QW * QW + 4 * E * RR + 2 * E * R1 +
                                             2 * (E + RD) * (E + RD) + 2 * E * E + E * R1 * E * R1);
    cudaFuncSetAttribute(k_iga_assemble<TB, RD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 grid(ceil_div(g.nb, TB), ceil_div(g.nb, TB));
    k_iga_assemble<TB, RD><<<grid, TB * TB, smem, s>>>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y, g.A);
}

// the load vector L (fp64, nb x nb) of mode 0 (saturation step) or 1 (projection of fq)
static void assemble(IgaDev &g, const float *S, const float *P, const float *K, const float *q, const float *fq,
                     int mode, float tau_phi, float mob, float grav_y, cudaStream_t s) {
    const long mm = (long)g.m * g.m, n2 = (long)g.nb * g.nb;
    if (assemble_split()) {
        k_iga_qp<<<ceil_div(mm, 256), 256, 0, s>>>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y);
        k_iga_gather<<<ceil_div(n2, 256), 256, 0, s>>>(g, g.A);
        return;
    }
    switch (g.r) {
        case 1: assemble_launch<16, 1>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y, s); break;
        case 2: assemble_launch<16, 2>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y, s); break;
        case 3: assemble_launch<16, 3>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y, s); break;
        case 4: assemble_launch<8, 4>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y, s); break;
        case 5: assemble_launch<8, 5>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y, s); break;
        default: assemble_launch<8, 6>(g, S, P, K, q, fq, mode, tau_phi, mob, grav_y, s); break;
    }
}

// X = M^-1 X along the row index, one thread per column; M = L D L^T with unit lower band L
__global__ void k_iga_band(IgaDev g, double *__restrict__ X) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g.nb) return;
    const int n = g.nb, r = g.r;
    for (int i = 0; i < n; ++i) {   // L z = x
        double v = X[(long)i * n + c];
        for (int d = 1; d <= r && d <= i; ++d) v = fma(-g.lf[i * r + d - 1], X[(long)(i - d) * n + c], v);
        X[(long)i * n + c] = v;
    }
    for (int i = 0; i < n; ++i) X[(long)i * n + c] *= g.dinv[i];
    for (int i = n - 1; i >= 0; --i) {   // L^T x = y
        double v = X[(long)i * n + c];
        for (int d = 1; d <= r && i + d < n; ++d) v = fma(-g.lf[(i + d) * r + d - 1], X[(long)(i + d) * n + c], v);
        X[(long)i * n + c] = v;
    }
}

__global__ void k_iga_transpose(const double *__restrict__ in, double *__restrict__ out, int n) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = by + y, c = bx + threadIdx.x;
        if (r < n && c < n) tile[y][threadIdx.x] = in[(long)r * n + c];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = bx + y, c = by + threadIdx.x;
        if (r < n && c < n) out[(long)r * n + c] = tile[threadIdx.x][y];
    }
}

__global__ void k_iga_dirichlet(double *X, int n) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    X[t] = 0.0;
    X[(long)(n - 1) * n + t] = 0.0;
    X[(long)t * n] = 0.0;
    X[(long)t * n + n - 1] = 0.0;
}

__global__ void k_iga_to_f32(const double *__restrict__ in, float *__restrict__ out, long n) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = (float)in[t];
}

// value and gradient of the field C at arbitrary points (device de Boor per point)
__global__ void k_iga_eval(IgaDev g, const float *__restrict__ C, const float *__restrict__ xy, long npts,
                           float *__restrict__ val, float *__restrict__ grad) {
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    const int r = g.r, ne = g.ne;
    float v[2][IGA_MAX_R + 1], d[2][IGA_MAX_R + 1];
    int i0[2];
    for (int ax = 0; ax < 2; ++ax) {
        const float x = fminf(fmaxf(xy[2 * p + ax], 0.f), 1.f);
        int e = min(max((int)floorf(x * ne), 0), ne - 1);
        const int span = e + r;
        auto knot = [&](int i) { return (float)min(max(i - r, 0), ne) / (float)ne; };
        float nd[IGA_MAX_R + 1][IGA_MAX_R + 1];
        float left[IGA_MAX_R + 1], right[IGA_MAX_R + 1];
        nd[0][0] = 1.f;
        for (int j = 1; j <= r; ++j) {
            left[j] = x - knot(span + 1 - j);
            right[j] = knot(span + j) - x;
            float saved = 0.f;
            for (int s = 0; s < j; ++s) {
                const float den = right[s + 1] + left[j - s];
                const float tmp = den != 0.f ? nd[j - 1][s] / den : 0.f;
                nd[j][s] = saved + right[s + 1] * tmp;
                saved = left[j - s] * tmp;
            }
            nd[j][j] = saved;
        }
        for (int a = 0; a <= r; ++a) {
            v[ax][a] = nd[r][a];
            const int i = span - r + a;
            float dd = 0.f;
            if (a >= 1) {
                const float den = knot(i + r) - knot(i);
                if (den > 0.f) dd += r * nd[r - 1][a - 1] / den;
            }
            if (a <= r - 1) {
                const float den = knot(i + r + 1) - knot(i + 1);
                if (den > 0.f) dd -= r * nd[r - 1][a] / den;
            }
            d[ax][a] = dd;
        }
        i0[ax] = span - r;
    }
    float s = 0.f, gx = 0.f, gy = 0.f;
    for (int b = 0; b <= r; ++b)
        for (int a = 0; a <= r; ++a) {
            const float c = C[(long)(i0[1] + b) * g.nb + i0[0] + a];
            s = fmaf(c, v[0][a] * v[1][b], s);
            gx = fmaf(c, d[0][a] * v[1][b], gx);
            gy = fmaf(c, v[0][a] * d[1][b], gy);
        }
    val[p] = s;
    if (grad) {
        grad[2 * p] = gx;
        grad[2 * p + 1] = gy;
    }
}

// The same solve with a block's 32 columns staged in shared memory: the substitutions are serial in
// i, so their latency (not bandwidth) bounds them, and shared memory has ~10x less of it than L2
constexpr int IGA_BAND_COLS = 32;
// a block's 32 columns -> shared memory [n][32], eight loads in flight per thread (a load-store
// loop keeps one: its global-load latency was most of the band kernels' time)
__device__ __forceinline__ void stage_cols(double *sx, const double *__restrict__ X, int n, int c0, int nc) {
    const int total = n * IGA_BAND_COLS, step = (int)blockDim.x;
    for (int e0 = threadIdx.x; e0 < total; e0 += 8 * step) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * step;
            const int i = e / IGA_BAND_COLS, cc = e % IGA_BAND_COLS;
            v[u] = (e < total && cc < nc) ? X[(long)i * n + c0 + cc] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (e0 + u * step < total) sx[e0 + u * step] = v[u];
    }
}

__global__ void k_iga_band_smem(IgaDev g, double *__restrict__ X) {
    extern __shared__ double sx[];   // [nb][IGA_BAND_COLS]
    const int n = g.nb, r = g.r;
    const int c0 = blockIdx.x * IGA_BAND_COLS;
    const int nc = min(IGA_BAND_COLS, n - c0);
    stage_cols(sx, X, n, c0, nc);
    __syncthreads();
    if (threadIdx.x < IGA_BAND_COLS) {
        double *col = sx + threadIdx.x;
        for (int i = 0; i < n; ++i) {   // L z = x
            double v = col[i * IGA_BAND_COLS];
            for (int d = 1; d <= r && d <= i; ++d) v = fma(-g.lf[i * r + d - 1], col[(i - d) * IGA_BAND_COLS], v);
            col[i * IGA_BAND_COLS] = v;
        }
        for (int i = 0; i < n; ++i) col[i * IGA_BAND_COLS] *= g.dinv[i];
        for (int i = n - 1; i >= 0; --i) {   // L^T x = D^-1 z
            double v = col[i * IGA_BAND_COLS];
            for (int d = 1; d <= r && i + d < n; ++d)
                v = fma(-g.lf[(i + d) * r + d - 1], col[(i + d) * IGA_BAND_COLS], v);
            col[i * IGA_BAND_COLS] = v;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * IGA_BAND_COLS; e += blockDim.x) {
        const int i = e / IGA_BAND_COLS, cc = e % IGA_BAND_COLS;
        if (cc < nc) X[(long)i * n + c0 + cc] = sx[e];
    }
}

// The substitutions with the band recurrence carried in registers: the last R values of the chain
// never go back through shared memory (its load-after-store latency set the step time of
// k_iga_band_smem); the band and 1/D are staged once per block (zero-padded, no bounds tests in the
// chain), and 1/D is folded into the forward pass.
template <int R>
__global__ void k_iga_band_reg(IgaDev g, double *__restrict__ X) {
    extern __shared__ double sx[];   // [nb][IGA_BAND_COLS] columns, [nb + R][R] band, [nb] 1/D
    const int n = g.nb;
    double *slf = sx + (size_t)n * IGA_BAND_COLS, *sdi = slf + (size_t)(n + R) * R;
    const int c0 = blockIdx.x * IGA_BAND_COLS;
    const int nc = min(IGA_BAND_COLS, n - c0);
    stage_cols(sx, X, n, c0, nc);
    for (int e = threadIdx.x; e < (n + R) * R; e += blockDim.x) {
        const int i = e / R, d = e % R + 1;
        slf[e] = (i < n && d <= i) ? g.lf[(long)i * g.r + d - 1] : 0.0;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sdi[i] = g.dinv[i];
    __syncthreads();
    if (threadIdx.x < IGA_BAND_COLS) {
        // U steps per batch: their loads are issued together, then the recurrence runs with one
        // DFMA on the critical path per step (the terms of older values are added first)
        constexpr int U = 8;
        double *col = sx + threadIdx.x;
        double z[R];
#pragma unroll
        for (int d = 0; d < R; ++d) z[d] = 0.0;
        for (int i0 = 0; i0 < n; i0 += U) {   // L z = x, then y = D^-1 z
            double xv[U], di[U], lv[U][R];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = min(i0 + u, n - 1);
                xv[u] = col[i * IGA_BAND_COLS];
                di[u] = sdi[i];
#pragma unroll
                for (int d = 0; d < R; ++d) lv[u][d] = slf[i * R + d];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                double v = xv[u];
#pragma unroll
                for (int d = R; d >= 1; --d) v = fma(-lv[u][d - 1], z[d - 1], v);
#pragma unroll
                for (int d = R - 1; d > 0; --d) z[d] = z[d - 1];
                z[0] = v;
                xv[u] = v * di[u];
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + u < n) col[(i0 + u) * IGA_BAND_COLS] = xv[u];
        }
#pragma unroll
        for (int d = 0; d < R; ++d) z[d] = 0.0;
        for (int i0 = n - 1; i0 >= 0; i0 -= U) {   // L^T x = y
            double yv[U], lv[U][R];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = max(i0 - u, 0);
                yv[u] = col[i * IGA_BAND_COLS];
#pragma unroll
                for (int d = 1; d <= R; ++d) lv[u][d - 1] = slf[(i + d) * R + d - 1];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                double v = yv[u];
#pragma unroll
                for (int d = R; d >= 1; --d) v = fma(-lv[u][d - 1], z[d - 1], v);
#pragma unroll
                for (int d = R - 1; d > 0; --d) z[d] = z[d - 1];
                z[0] = v;
                yv[u] = v;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 - u >= 0) col[(i0 - u) * IGA_BAND_COLS] = yv[u];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * IGA_BAND_COLS; e += blockDim.x) {
        const int i = e / IGA_BAND_COLS, cc = e % IGA_BAND_COLS;
        if (cc < nc) X[(long)i * n + c0 + cc] = sx[e];
    }
}

// The substitutions of k_iga_band_reg split along the chain: NSEG segments of every column run at
// once. A substitution is linear, so a segment's values are its particular solution from a zero
// entry state (phase A) plus the response to the true entry state (the R values before it; phase
// C), whose coefficients (cfw / cbw, the homogeneous solutions inside the segment) depend only on
// the mass matrix and are precomputed in fp64 at create. Only the entry states are carried from
// segment to segment, one short step per segment (phase B). 1028 dependent steps per column become
// 2 x (n / NSEG + NSEG).
// TR = false: the block's 32 columns of X (solve along the row index); TR = true: 32 rows of X (solve
// along the column index, X^T staged on the fly: no transposes around the second direction)
template <int R, bool TR>
__global__ void k_iga_band_seg(IgaDev g, double *__restrict__ X) {
    constexpr int CS = TR ? IGA_BAND_COLS + 1 : IGA_BAND_COLS;   // odd stride: the transposed staging is conflict-light
    extern __shared__ double sx[];   // [nb][32] columns, [nb + R][R] band, [nb] 1/D, [nseg][R][32] entry
                                     // states, [nb][R] forward and backward responses
    const int n = g.nb, S = g.nseg;
    double *slf = sx + (size_t)n * CS, *sdi = slf + (size_t)(n + R) * R;
    double *sst = sdi + n;
    double *scf = sst + (size_t)S * R * IGA_BAND_COLS, *scb = scf + (size_t)n * R;
    for (int e = threadIdx.x; e < n * R; e += blockDim.x) {   // (global loads in phase B were its latency)
        scf[e] = g.cfw[e];
        scb[e] = g.cbw[e];
    }
    const int c0 = blockIdx.x * IGA_BAND_COLS;
    const int nc = min(IGA_BAND_COLS, n - c0);
    if (TR) {
        const int total = n * IGA_BAND_COLS, step = (int)blockDim.x;
        for (int e0 = threadIdx.x; e0 < total; e0 += 8 * step) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * step, cc = e / n, i = e % n;
                v[u] = (e < total && cc < nc) ? X[(long)(c0 + cc) * n + i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * step;
                if (e < total) sx[(e % n) * CS + e / n] = v[u];
            }
        }
    } else {
        stage_cols(sx, X, n, c0, nc);
    }
    for (int e = threadIdx.x; e < (n + R) * R; e += blockDim.x) {
        const int i = e / R, d = e % R + 1;
        slf[e] = (i < n && d <= i) ? g.lf[(long)i * g.r + d - 1] : 0.0;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sdi[i] = g.dinv[i];
    __syncthreads();
    const int col = threadIdx.x % IGA_BAND_COLS, sg = threadIdx.x / IGA_BAND_COLS;
    const bool act = sg < S;
    const int a = act ? g.seg0[sg] : 0, b = act ? g.seg0[sg + 1] : 0;
    double *cx = sx + col;
    // ---- forward: L z = x from a zero entry state
    if (act) {
        double z[R];
#pragma unroll
        for (int d = 0; d < R; ++d) z[d] = 0.0;
        for (int i = a; i < b; ++i) {
            double v = cx[i * CS];
#pragma unroll
            for (int d = R; d >= 1; --d) v = fma(-slf[i * R + d - 1], z[d - 1], v);
#pragma unroll
            for (int d = R - 1; d > 0; --d) z[d] = z[d - 1];
            z[0] = v;
            cx[i * CS] = v;
        }
    }
    __syncthreads();
    if (sg == 0) {   // entry states: st_s[c] = z_{a_s - 1 - c}
        double st[R];
#pragma unroll
        for (int c = 0; c < R; ++c) st[c] = 0.0;
        for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
            for (int c = 0; c < R; ++c) sst[((size_t)s2 * R + c) * IGA_BAND_COLS + col] = st[c];
            if (s2 + 1 == S) break;
            const int e2 = g.seg0[s2 + 1];
            double nx[R];
#pragma unroll
            for (int c = 0; c < R; ++c) {
                const int j = e2 - 1 - c;
                double v = cx[j * CS];
#pragma unroll
                for (int c2 = 0; c2 < R; ++c2) v = fma(scf[j * R + c2], st[c2], v);
                nx[c] = v;
            }
#pragma unroll
            for (int c = 0; c < R; ++c) st[c] = nx[c];
        }
    }
    __syncthreads();
    if (act) {   // z = particular + response to the entry state, then y = D^-1 z
        double st[R];
#pragma unroll
        for (int c = 0; c < R; ++c) st[c] = sst[((size_t)sg * R + c) * IGA_BAND_COLS + col];
        for (int i = a; i < b; ++i) {
            double v = cx[i * CS];
#pragma unroll
            for (int c = 0; c < R; ++c) v = fma(scf[i * R + c], st[c], v);
            cx[i * CS] = v * sdi[i];
        }
    }
    __syncthreads();
    // ---- backward: L^T x = y from a zero exit state
    if (act) {
        double z[R];
#pragma unroll
        for (int d = 0; d < R; ++d) z[d] = 0.0;
        for (int i = b - 1; i >= a; --i) {
            double v = cx[i * CS];
#pragma unroll
            for (int d = R; d >= 1; --d) v = fma(-slf[(i + d) * R + d - 1], z[d - 1], v);
#pragma unroll
            for (int d = R - 1; d > 0; --d) z[d] = z[d - 1];
            z[0] = v;
            cx[i * CS] = v;
        }
    }
    __syncthreads();
    if (sg == 0) {   // exit states: st_s[c] = x_{b_s + c}
        double st[R];
#pragma unroll
        for (int c = 0; c < R; ++c) st[c] = 0.0;
        for (int s2 = S - 1; s2 >= 0; --s2) {
#pragma unroll
            for (int c = 0; c < R; ++c) sst[((size_t)s2 * R + c) * IGA_BAND_COLS + col] = st[c];
            if (s2 == 0) break;
            const int e2 = g.seg0[s2];
            double nx[R];
#pragma unroll
            for (int c = 0; c < R; ++c) {
                const int j = e2 + c;
                double v = cx[j * CS];
#pragma unroll
                for (int c2 = 0; c2 < R; ++c2) v = fma(scb[j * R + c2], st[c2], v);
                nx[c] = v;
            }
#pragma unroll
            for (int c = 0; c < R; ++c) st[c] = nx[c];
        }
    }
    __syncthreads();
    if (act) {
        double st[R];
#pragma unroll
        for (int c = 0; c < R; ++c) st[c] = sst[((size_t)sg * R + c) * IGA_BAND_COLS + col];
        for (int i = a; i < b; ++i) {
            double v = cx[i * CS];
#pragma unroll
            for (int c = 0; c < R; ++c) v = fma(scb[i * R + c], st[c], v);
            cx[i * CS] = v;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * IGA_BAND_COLS; e += blockDim.x) {
        if (TR) {
            const int cc = e / n, i = e % n;
            if (cc < nc) X[(long)(c0 + cc) * n + i] = sx[i * CS + cc];
        } else {
            const int i = e / IGA_BAND_COLS, cc = e % IGA_BAND_COLS;
            if (cc < nc) X[(long)i * n + c0 + cc] = sx[e];
        }
    }
}

template <int R>
static size_t band_seg_smem(int n, int nseg) {
    return sizeof(double) * ((size_t)n * (IGA_BAND_COLS + 1) + (size_t)(n + R) * R + n + (size_t)nseg * R * IGA_BAND_COLS +
                             2 * (size_t)n * R);
}

template <int R>
static bool band_seg_launch(IgaDev &g, double *X, bool tr, cudaStream_t s) {
    const size_t smem = band_seg_smem<R>(g.nb, g.nseg);
    if (g.nseg < 2 || smem > 200 * 1024) return false;
    const dim3 grid(ceil_div(g.nb, IGA_BAND_COLS)), block(IGA_BAND_COLS * g.nseg);
    if (tr) {
        cudaFuncSetAttribute(k_iga_band_seg<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        k_iga_band_seg<R, true><<<grid, block, smem, s>>>(g, X);
    } else {
        cudaFuncSetAttribute(k_iga_band_seg<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        k_iga_band_seg<R, false><<<grid, block, smem, s>>>(g, X);
    }
    return true;
}

static bool band_seg_ok(const IgaDev &g) {
    const char *bv = getenv("CRVPINN_IGA_BAND");   // tuning knob: "reg" / "smem" = the serial kernels
    if (bv && (strcmp(bv, "reg") == 0 || strcmp(bv, "smem") == 0)) return false;
    if (g.nseg < 2) return false;
    size_t sm;
    switch (g.r) {
        case 1: sm = band_seg_smem<1>(g.nb, g.nseg); break;
        case 2: sm = band_seg_smem<2>(g.nb, g.nseg); break;
        case 3: sm = band_seg_smem<3>(g.nb, g.nseg); break;
        case 4: sm = band_seg_smem<4>(g.nb, g.nseg); break;
        case 5: sm = band_seg_smem<5>(g.nb, g.nseg); break;
        default: sm = band_seg_smem<6>(g.nb, g.nseg); break;
    }
    return sm <= 200 * 1024;
}

static bool band_seg(IgaDev &g, double *X, bool tr, cudaStream_t s) {
    switch (g.r) {
        case 1: return band_seg_launch<1>(g, X, tr, s);
        case 2: return band_seg_launch<2>(g, X, tr, s);
        case 3: return band_seg_launch<3>(g, X, tr, s);
        case 4: return band_seg_launch<4>(g, X, tr, s);
        case 5: return band_seg_launch<5>(g, X, tr, s);
        default: return band_seg_launch<6>(g, X, tr, s);
    }
}

template <int R>
static size_t band_reg_smem(int n) { return sizeof(double) * ((size_t)n * IGA_BAND_COLS + (size_t)(n + R) * R + n); }

template <int R>
static bool band_reg_launch(IgaDev &g, double *X, cudaStream_t s) {
    const size_t smem = band_reg_smem<R>(g.nb);
    if (smem > 200 * 1024) return false;
    // per device and cheap: set on every call (a process may use several devices)
    cudaFuncSetAttribute(k_iga_band_reg<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_iga_band_reg<R><<<ceil_div(g.nb, IGA_BAND_COLS), 256, smem, s>>>(g, X);
    return true;
}

static bool band_reg(IgaDev &g, double *X, cudaStream_t s) {
    switch (g.r) {
        case 1: return band_reg_launch<1>(g, X, s);
        case 2: return band_reg_launch<2>(g, X, s);
        case 3: return band_reg_launch<3>(g, X, s);
        case 4: return band_reg_launch<4>(g, X, s);
        case 5: return band_reg_launch<5>(g, X, s);
        default: return band_reg_launch<6>(g, X, s);
    }
}

// L -> C = M^-1 L M^-1 (both directions), in place in g.A (g.B scratch)
void kron_solve(IgaDev &g, cudaStream_t s) {
    const int n = g.nb;
    const dim3 tb(32, 8), tg((n + 31) / 32, (n + 31) / 32);
    const size_t smem = sizeof(double) * (size_t)n * IGA_BAND_COLS;
    const char *bv = getenv("CRVPINN_IGA_BAND");   // tuning knob: "smem" = k_iga_band_smem
    const bool reg = !(bv && strcmp(bv, "smem") == 0) && band_reg_smem<6>(n) <= 200 * 1024;
    if (band_seg_ok(g)) {
        band_seg(g, g.A, false, s);   // along l (rows)
        band_seg(g, g.A, true, s);    // along k, in place: the result is already in g.A
        return;
    } else if (reg) {
        band_reg(g, g.A, s);                       // along l (rows)
        k_iga_transpose<<<tg, tb, 0, s>>>(g.A, g.B, n);
        band_reg(g, g.B, s);                       // along k
    } else if (smem <= 200 * 1024) {
        // per device and cheap: set on every call (a process may use several devices)
        cudaFuncSetAttribute(k_iga_band_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        k_iga_band_smem<<<ceil_div(n, IGA_BAND_COLS), 256, smem, s>>>(g, g.A);   // along l (rows)
        k_iga_transpose<<<tg, tb, 0, s>>>(g.A, g.B, n);
        k_iga_band_smem<<<ceil_div(n, IGA_BAND_COLS), 256, smem, s>>>(g, g.B);   // along k
    } else {   // very large spaces: straight from global memory
        k_iga_band<<<ceil_div(n, 128), 128, 0, s>>>(g, g.A);
        k_iga_transpose<<<tg, tb, 0, s>>>(g.A, g.B, n);
        k_iga_band<<<ceil_div(n, 128), 128, 0, s>>>(g, g.B);
    }
    k_iga_transpose<<<tg, tb, 0, s>>>(g.B, g.A, n);
}

}  // namespace
}  // namespace crv

// ================================================================ C ABI
struct crvpinn_iga {
    crv::IgaDev g;
    int device = 0;
    std::string err;
};

using crv::IgaDev;

static int iga_fail(crvpinn_iga *h, int code, const std::string &m) {
    if (h) h->err = m;
    return code;
}
#define IGA_CK(call)                                                                      \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) return iga_fail(h, CRVPINN_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

static int iga_stage(crvpinn_iga *h, size_t floats) {
    IgaDev &g = h->g;
    if (floats <= g.io_cap) return CRVPINN_OK;
    if (g.io) cudaFree(g.io);
    g.io = nullptr;
    g.io_cap = 0;
    IGA_CK(cudaMalloc(&g.io, sizeof(float) * floats));
    g.io_cap = floats;
    return CRVPINN_OK;
}

extern "C" {

int crvpinn_iga_create(crvpinn_iga **out, int n_elements, int degree, int device) {
    if (!out) return CRVPINN_EINVAL;
    *out = nullptr;
    if (n_elements < 1 || n_elements > 8192 || degree < 1 || degree > crv::IGA_MAX_R) return CRVPINN_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) return CRVPINN_ECUDA;
    crvpinn_iga *h = new crvpinn_iga();
    h->device = device;
    if (cudaSetDevice(device) != cudaSuccess) { delete h; return CRVPINN_ECUDA; }
    IgaDev &g = h->g;
    g.ne = n_elements; g.r = degree; g.nb = n_elements + degree; g.m = n_elements * (degree + 1);
    const int R1 = degree + 1, nb = g.nb;
    std::vector<double> gx, gw;
    crv::gauss01(R1, gx, gw);
    std::vector<float> bv((size_t)g.ne * R1 * R1), bd(bv.size()), w((size_t)g.m);
    std::vector<double> mass((size_t)nb * (degree + 1), 0.0);   // mass[i][d] = M_{i, i+d}, d = 0..r
    std::vector<double> val(R1), der(R1);
    for (int e = 0; e < g.ne; ++e)
        for (int q = 0; q < R1; ++q) {
            const double x = (e + gx[q]) / g.ne, wq = gw[q] / g.ne;
            const int i0 = crv::bspline_local(g.ne, degree, x, val.data(), der.data());
            for (int a = 0; a < R1; ++a) {
                bv[((size_t)e * R1 + q) * R1 + a] = (float)val[a];
                bd[((size_t)e * R1 + q) * R1 + a] = (float)der[a];
                for (int b = a; b < R1; ++b) mass[(size_t)(i0 + a) * R1 + (b - a)] += wq * val[a] * val[b];
            }
            w[(size_t)e * R1 + q] = (float)wq;
        }
    // banded LDL^T of the SPD mass matrix, fp64: lf[i][d-1] = L_{i,i-d}
    std::vector<double> Lb((size_t)nb * degree, 0.0), D(nb, 0.0);
    for (int i = 0; i < nb; ++i) {
        for (int d = degree; d >= 1; --d) {   // L_{i,j}, j = i - d
            const int j = i - d;
            if (j < 0) continue;
            double v = mass[(size_t)j * R1 + d];   // M_{j,i}
            for (int t = 1; t <= degree && j - t >= 0; ++t) {
                const int dl = i - (j - t);        // L_{i, j-t}
                if (dl <= degree) v -= Lb[(size_t)i * degree + dl - 1] * Lb[(size_t)j * degree + t - 1] * D[j - t];
            }
            Lb[(size_t)i * degree + d - 1] = v / D[j];
        }
        double v = mass[(size_t)i * R1 + 0];
        for (int d = 1; d <= degree && i - d >= 0; ++d) {
            const double l = Lb[(size_t)i * degree + d - 1];
            v -= l * l * D[i - d];
        }
        D[i] = v;
    }
    std::vector<double> lf(Lb), dinv(nb);
    for (int i = 0; i < nb; ++i) dinv[i] = 1.0 / D[i];
    // chain segments of k_iga_band_seg (balanced, each >= max(degree, 8) rows) and the homogeneous
    // responses of both substitutions to a segment's entry state
    int nseg = nb / 32 > 0 ? (nb + 31) / 32 : 1;
    if (nseg > 32) nseg = 32;
    while (nseg > 1 && nb / nseg < (degree > 8 ? degree : 8)) --nseg;
    std::vector<int> seg0(nseg + 1);
    for (int s2 = 0; s2 <= nseg; ++s2) seg0[s2] = (int)((long)s2 * nb / nseg);
    std::vector<double> cfw((size_t)nb * degree, 0.0), cbw((size_t)nb * degree, 0.0);
    for (int s2 = 0; s2 < nseg; ++s2) {
        const int a = seg0[s2], b = seg0[s2 + 1];
        for (int c = 0; c < degree; ++c) {
            std::vector<double> z((size_t)(b - a + degree), 0.0);   // z[degree + (i - a)]; entry z[degree-1-c] = 1
            z[(size_t)(degree - 1 - c)] = 1.0;
            for (int i = a; i < b; ++i) {
                double v = 0.0;
                for (int d = 1; d <= degree; ++d)
                    if (i - d >= 0) v -= Lb[(size_t)i * degree + d - 1] * z[(size_t)(degree + i - a - d)];
                z[(size_t)(degree + i - a)] = v;
                cfw[(size_t)i * degree + c] = v;
            }
            std::vector<double> x((size_t)(b - a + degree), 0.0);   // x[i - a]; exit x[b - a + c] = 1
            x[(size_t)(b - a + c)] = 1.0;
            for (int i = b - 1; i >= a; --i) {
                double v = 0.0;
                for (int d = 1; d <= degree; ++d)
                    if (i + d < nb) v -= Lb[(size_t)(i + d) * degree + d - 1] * x[(size_t)(i - a + d)];
                x[(size_t)(i - a)] = v;
                cbw[(size_t)i * degree + c] = v;
            }
        }
    }
    g.nseg = nseg;
    const long mm = (long)g.m * g.m;
    bool ok = cudaMalloc(&g.bv, sizeof(float) * bv.size()) == cudaSuccess &&
              cudaMalloc(&g.bd, sizeof(float) * bd.size()) == cudaSuccess &&
              cudaMalloc(&g.gw, sizeof(float) * w.size()) == cudaSuccess &&
              cudaMalloc(&g.lf, sizeof(double) * (lf.size() ? lf.size() : 1)) == cudaSuccess &&
              cudaMalloc(&g.dinv, sizeof(double) * nb) == cudaSuccess &&
              cudaMalloc(&g.seg0, sizeof(int) * seg0.size()) == cudaSuccess &&
              cudaMalloc(&g.cfw, sizeof(double) * cfw.size()) == cudaSuccess &&
              cudaMalloc(&g.cbw, sizeof(double) * cbw.size()) == cudaSuccess &&
              cudaMalloc(&g.qv, sizeof(float) * 3 * mm) == cudaSuccess &&
              cudaMalloc(&g.A, sizeof(double) * nb * nb) == cudaSuccess &&
              cudaMalloc(&g.B, sizeof(double) * nb * nb) == cudaSuccess &&
              cudaMalloc(&g.outf, sizeof(float) * nb * nb) == cudaSuccess &&
              cudaEventCreate(&g.e0) == cudaSuccess && cudaEventCreate(&g.e1) == cudaSuccess;
    if (ok)
        ok = cudaMemcpy(g.bv, bv.data(), sizeof(float) * bv.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(g.bd, bd.data(), sizeof(float) * bd.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(g.gw, w.data(), sizeof(float) * w.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(g.lf, lf.data(), sizeof(double) * lf.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(g.dinv, dinv.data(), sizeof(double) * nb, cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(g.seg0, seg0.data(), sizeof(int) * seg0.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(g.cfw, cfw.data(), sizeof(double) * cfw.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(g.cbw, cbw.data(), sizeof(double) * cbw.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
        crvpinn_iga_destroy(h);
        return CRVPINN_ENOMEM;
    }
    *out = h;
    return CRVPINN_OK;
}

int crvpinn_iga_num_basis(const crvpinn_iga *h) { return h ? h->g.nb : 0; }

long crvpinn_iga_num_quad_points(const crvpinn_iga *h) { return h ? (long)h->g.m * h->g.m : 0; }

int crvpinn_iga_quad_points(crvpinn_iga *h, float *xy) {
    if (!h || !xy) return iga_fail(h, CRVPINN_EINVAL, "null argument");
    const int R1 = h->g.r + 1;
    std::vector<double> gx, gw;
    crv::gauss01(R1, gx, gw);
    const int m = h->g.m;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
            const long p = (long)j * m + i;
            xy[2 * p] = (float)((i / R1 + gx[i % R1]) / h->g.ne);
            xy[2 * p + 1] = (float)((j / R1 + gx[j % R1]) / h->g.ne);
        }
    return CRVPINN_OK;
}

int crvpinn_iga_project(crvpinn_iga *h, const float *fq, float *coef) {
    if (!h || !fq || !coef) return iga_fail(h, CRVPINN_EINVAL, "null argument");
    IgaDev &g = h->g;
    IGA_CK(cudaSetDevice(h->device));
    const long mm = (long)g.m * g.m, n2 = (long)g.nb * g.nb;
    int rc = iga_stage(h, (size_t)mm);
    if (rc) return rc;
    IGA_CK(cudaMemcpy(g.io, fq, sizeof(float) * mm, cudaMemcpyHostToDevice));
    cudaEventRecord(g.e0, 0);
    crv::assemble(g, nullptr, nullptr, nullptr, nullptr, g.io, 1, 0.f, 0.f, 0.f, 0);
    crv::kron_solve(g, 0);
    crv::k_iga_to_f32<<<crv::ceil_div(n2, 256), 256>>>(g.A, g.outf, n2);
    cudaEventRecord(g.e1, 0);
    IGA_CK(cudaMemcpy(coef, g.outf, sizeof(float) * n2, cudaMemcpyDeviceToHost));
    IGA_CK(cudaGetLastError());
    cudaEventElapsedTime(&g.last_ms, g.e0, g.e1);
    return CRVPINN_OK;
}

int crvpinn_iga_saturation_step(crvpinn_iga *h, const float *S, const float *P, const float *K_elem,
                                const float *q_elem, double tau, double phi, double mobility_ratio,
                                double density_ratio, double gravity, float *S_out) {
    if (!h || !S || !P || !K_elem || !q_elem || !S_out) return iga_fail(h, CRVPINN_EINVAL, "null argument");
    if (!(tau >= 0.0) || !(phi > 0.0) || !std::isfinite(mobility_ratio) || !std::isfinite(density_ratio) ||
        !std::isfinite(gravity))
        return iga_fail(h, CRVPINN_EINVAL, "need tau >= 0, phi > 0 and finite parameters");
    IgaDev &g = h->g;
    IGA_CK(cudaSetDevice(h->device));
    const long n2 = (long)g.nb * g.nb, ne2 = (long)g.ne * g.ne;
    int rc = iga_stage(h, (size_t)(2 * n2 + 2 * ne2));
    if (rc) return rc;
    float *dS = g.io, *dP = g.io + n2, *dK = g.io + 2 * n2, *dq = g.io + 2 * n2 + ne2;
    IGA_CK(cudaMemcpy(dS, S, sizeof(float) * n2, cudaMemcpyHostToDevice));
    IGA_CK(cudaMemcpy(dP, P, sizeof(float) * n2, cudaMemcpyHostToDevice));
    IGA_CK(cudaMemcpy(dK, K_elem, sizeof(float) * ne2, cudaMemcpyHostToDevice));
    IGA_CK(cudaMemcpy(dq, q_elem, sizeof(float) * ne2, cudaMemcpyHostToDevice));
    cudaEventRecord(g.e0, 0);
    crv::assemble(g, dS, dP, dK, dq, nullptr, 0, (float)(tau / phi), (float)mobility_ratio,
                  (float)(density_ratio * gravity), 0);
    crv::kron_solve(g, 0);
    crv::k_iga_dirichlet<<<crv::ceil_div(g.nb, 256), 256>>>(g.A, g.nb);
    crv::k_iga_to_f32<<<crv::ceil_div(n2, 256), 256>>>(g.A, g.outf, n2);
    cudaEventRecord(g.e1, 0);
    IGA_CK(cudaMemcpy(S_out, g.outf, sizeof(float) * n2, cudaMemcpyDeviceToHost));
    IGA_CK(cudaGetLastError());
    cudaEventElapsedTime(&g.last_ms, g.e0, g.e1);
    return CRVPINN_OK;
}

int crvpinn_iga_eval(crvpinn_iga *h, const float *coef, long n, const float *xy, float *val, float *grad) {
    if (!h || n < 0) return iga_fail(h, CRVPINN_EINVAL, "bad argument");
    if (n == 0) return CRVPINN_OK;
    if (!coef || !xy || !val) return iga_fail(h, CRVPINN_EINVAL, "null argument");
    IgaDev &g = h->g;
    IGA_CK(cudaSetDevice(h->device));
    const long n2 = (long)g.nb * g.nb;
    int rc = iga_stage(h, (size_t)(n2 + 5 * n));
    if (rc) return rc;
    float *dC = g.io, *dxy = g.io + n2, *dv = dxy + 2 * n, *dg = dv + n;
    IGA_CK(cudaMemcpy(dC, coef, sizeof(float) * n2, cudaMemcpyHostToDevice));
    IGA_CK(cudaMemcpy(dxy, xy, sizeof(float) * 2 * n, cudaMemcpyHostToDevice));
    crv::k_iga_eval<<<crv::ceil_div(n, 256), 256>>>(g, dC, dxy, n, dv, grad ? dg : nullptr);
    IGA_CK(cudaMemcpy(val, dv, sizeof(float) * n, cudaMemcpyDeviceToHost));
    if (grad) IGA_CK(cudaMemcpy(grad, dg, sizeof(float) * 2 * n, cudaMemcpyDeviceToHost));
    IGA_CK(cudaGetLastError());
    return CRVPINN_OK;
}

double crvpinn_iga_last_ms(const crvpinn_iga *h) { return h ? (double)h->g.last_ms : 0.0; }

const char *crvpinn_iga_last_error(const crvpinn_iga *h) { return h ? h->err.c_str() : ""; }

void crvpinn_iga_destroy(crvpinn_iga *h) {
    if (!h) return;
    IgaDev &g = h->g;
    cudaSetDevice(h->device);
    void *bufs[] = {g.bv, g.bd, g.gw, g.lf, g.dinv, g.seg0, g.cfw, g.cbw, g.qv, g.A, g.B, g.io, g.outf};
    for (void *p : bufs)
        if (p) cudaFree(p);
    if (g.e0) cudaEventDestroy(g.e0);
    if (g.e1) cudaEventDestroy(g.e1);
    delete h;
}

}  // extern "C"
