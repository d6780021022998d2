"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Each test names the pin (P1..P13) and the passage it follows. None of these re-calls the
oracle's own formula as its reference: the references are closed forms, brute-force literal
definitions, finite differences, eigen-decompositions, or independent library routines
(numpy/scipy dense solves, torch autograd, torch.optim.Adam).

Inputs are fp32 (the ABI's input type) promoted to fp64, so closed forms that involve the
source f hold to fp32 input rounding (~1e-7 relative), not to 1e-15.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _ctx(N, widths=(2, 8, 1), K=None, S=None, f=None, theta=None, **kw):
    nn = (N + 1) ** 2
    K = np.ones(nn, np.float32) if K is None else K
    S = np.zeros(nn, np.float32) if S is None else S
    f = np.zeros(nn, np.float32) if f is None else f
    return oracle.Oracle(N, widths, K, S, f, theta, **kw)


def _dst_matrix(N):
    n = N - 1
    i = np.arange(1, n + 1)
    S = math.sqrt(2.0 / N) * np.sin(math.pi * np.outer(i, i) / N)
    lam = 4.0 * np.sin(math.pi * i / (2.0 * N)) ** 2
    return S, lam


def _gram_inv_dst(N, R):
    """G^-1 R via the 2-D sine eigenbasis of the 5-point matrix (independent of the LU)."""
    S, lam = _dst_matrix(N)
    h = 1.0 / N
    n = N - 1
    Rm = R.reshape(n, n)
    Z = (S @ Rm @ S) / (lam[:, None] + lam[None, :])
    return (h * h * (S @ Z @ S)).reshape(-1)


# --------------------------------------------------------------------------- P0: Table 1
def test_table1_golden_mobility_ratio():
    """Reading R10: M = mu_w/mu_g from Table 1 (golden fixture)."""
    with open(os.path.join(GOLDEN, "table1.json")) as fh:
        t1 = json.load(fh)
    assert t1["mu_w"] == 25.35e-5 and t1["mu_g"] == 3.95e-5
    assert abs(oracle.MOBILITY_RATIO - t1["mu_w"] / t1["mu_g"]) < 1e-15
    assert abs(W.MOBILITY_RATIO - 6.417721518987342) < 1e-12


def test_alpha_A0_special_cases():
    """alpha = K((1-S) + M S): S=0 -> K, S=1 -> M K, clamping of S."""
    N = 4
    nn = (N + 1) ** 2
    rng = np.random.default_rng(3)
    K = rng.uniform(0.5, 2.0, nn).astype(np.float32)
    for s, factor in [(0.0, 1.0), (1.0, oracle.MOBILITY_RATIO), (-0.3, 1.0), (1.7, oracle.MOBILITY_RATIO)]:
        o = _ctx(N, K=K, S=np.full(nn, s, np.float32))
        np.testing.assert_allclose(o.alpha(), K.astype(np.float64) * factor, rtol=1e-15)
    # monotone in S when mu_g < mu_w
    Ss = np.linspace(0, 1, 100).astype(np.float32)
    o = _ctx(N, K=np.ones(nn, np.float32), S=np.resize(Ss, nn))
    a = o.alpha()[:100]
    assert np.all(np.diff(a) > 0)


# --------------------------------------------------------------------------- P1, P2: Gram
@pytest.mark.parametrize("N", [3, 4, 7, 10])
def test_P1_gram_matrix_entries(N):
    """G entries (Eq. 26): 4h^-2 diagonal, -h^-2 for 4-neighbours, 0 else.

    Probed through the oracle's matvec on unit vectors; the reference is the neighbour rule
    in (i,j) lattice coordinates, not the oracle's row-offset arithmetic.
    """
    o = _ctx(N, factor_gram=False)
    n, h2i = N - 1, float(N * N)
    for col in range(n * n):
        e = np.zeros(n * n)
        e[col] = 1.0
        g = o.gram_matvec(e)
        ci, cj = col % n, col // n
        for row in range(n * n):
            ri, rj = row % n, row // n
            d = abs(ri - ci) + abs(rj - cj)
            want = 4 * h2i if d == 0 else (-h2i if d == 1 else 0.0)
            assert abs(g[row] - want) <= 1e-14 * h2i


@pytest.mark.parametrize("N", [4, 6, 8])
def test_P2_gram_solve_vs_dense_lapack(N):
    """LU substitution (Eq. 28) == dense LAPACK solve of G at N<=8 to 1e-12."""
    o = _ctx(N)
    n = N - 1
    G = np.column_stack([o.gram_matvec(np.eye(n * n)[:, c]) for c in range(n * n)])
    rng = np.random.default_rng(N)
    for _ in range(3):
        r = rng.standard_normal(n * n)
        np.testing.assert_allclose(o.gram_solve(r), np.linalg.solve(G, r), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("N", [8, 16, 33])
def test_P2_gram_solve_eigenpairs(N):
    """G^-1 phi_ab = h^2/(lam_a+lam_b) phi_ab, phi_ab = sin(pi a i/N) sin(pi b j/N) (closed form)."""
    o = _ctx(N)
    n, h = N - 1, 1.0 / N
    i = np.arange(1, n + 1)
    for a, b in [(1, 1), (2, 5), (n, 1), (n // 2, n)]:
        phi = np.outer(np.sin(math.pi * b * i / N), np.sin(math.pi * a * i / N)).reshape(-1)
        lam = 4 * math.sin(math.pi * a / (2 * N)) ** 2 + 4 * math.sin(math.pi * b / (2 * N)) ** 2
        np.testing.assert_allclose(o.gram_solve(phi), h * h / lam * phi, rtol=1e-11, atol=1e-13)


def test_P2_gram_solve_vs_dst_random():
    """Band LU solve == 2-D sine-transform solve on random RES (N=32)."""
    N = 32
    o = _ctx(N)
    r = np.random.default_rng(0).standard_normal((N - 1) ** 2)
    np.testing.assert_allclose(o.gram_solve(r), _gram_inv_dst(N, r), rtol=1e-11, atol=1e-15)


# --------------------------------------------------------------------------- P3: stencil
def _literal_residual(N, alpha, u, f):
    """Eq. 25 by brute force: h^2 sum_{p in Omega_h} alpha_p grad+u_p . grad+delta_kl(p) - h^2 f_kl.

    Full sums over every lattice node p (no use of the delta's support); grad+ (Eq. 22) of any
    lattice function is taken as 0 where the forward neighbour leaves the lattice.
    """
    h = 1.0 / N
    A = alpha.reshape(N + 1, N + 1)
    U = u.reshape(N + 1, N + 1)

    def grad_plus(F):
        gx = np.zeros_like(F)
        gy = np.zeros_like(F)
        gx[:, :-1] = (F[:, 1:] - F[:, :-1]) / h
        gy[:-1, :] = (F[1:, :] - F[:-1, :]) / h
        return gx, gy

    ux, uy = grad_plus(U)
    # grad+ u at i=N or j=N is never paired with a non-zero grad+ delta for interior tests
    out = np.zeros((N - 1) * (N - 1))
    for l in range(1, N):
        for k in range(1, N):
            D = np.zeros((N + 1, N + 1))
            D[l, k] = 1.0
            dx, dy = grad_plus(D)
            lhs = h * h * np.sum(A * (ux * dx + uy * dy))
            rhs = h * h * np.sum(f.reshape(N + 1, N + 1) * D)
            out[(l - 1) * (N - 1) + (k - 1)] = lhs - rhs
    return out


@pytest.mark.parametrize("N", [4, 7, 8])
def test_P3_residual_vs_literal_inner_product(N):
    K, S, f = W.random_fields(N, seed=N)
    o = _ctx(N, K=K, S=S, f=f, factor_gram=False)
    u = np.random.default_rng(N + 1).standard_normal((N + 1) ** 2)
    u = u.reshape(N + 1, N + 1)
    u[0, :] = u[-1, :] = u[:, 0] = u[:, -1] = 0.0
    u = u.reshape(-1)
    want = _literal_residual(N, o.alpha(), u, f.astype(np.float64))
    np.testing.assert_allclose(o.residual(u), want, rtol=1e-12, atol=1e-13)


def test_residual_special_cases():
    """alpha=1 collapses to the 5-point Laplacian; u=0, f=1 gives RES = -h^2."""
    N = 8
    nn = (N + 1) ** 2
    o = _ctx(N, f=np.ones(nn, np.float32), factor_gram=False)
    np.testing.assert_array_equal(o.residual(np.zeros(nn)), np.full((N - 1) ** 2, -1.0 / N ** 2))
    o0 = _ctx(N, factor_gram=False)
    u = np.random.default_rng(1).standard_normal((N + 1, N + 1))
    u[0, :] = u[-1, :] = u[:, 0] = u[:, -1] = 0.0
    lap = 4 * u[1:-1, 1:-1] - u[1:-1, :-2] - u[1:-1, 2:] - u[:-2, 1:-1] - u[2:, 1:-1]
    np.testing.assert_allclose(o0.residual(u.reshape(-1)), lap.reshape(-1), rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------------------- P4, P5: closed forms
def test_P4_residual_zero_manufactured_sine():
    """alpha=1, f=2 pi^2 sin sin: u = c_h sin sin solves the discrete equation exactly (reading R1)."""
    N = 32
    h = 1.0 / N
    X, Y = W.grid_xy(N)
    f = (2 * math.pi ** 2 * np.sin(math.pi * X) * np.sin(math.pi * Y)).astype(np.float32)
    o = _ctx(N, f=f.reshape(-1))
    ch = (math.pi * h / 2) ** 2 / math.sin(math.pi * h / 2) ** 2
    assert abs(ch - 1.000803577679372) < 1e-14
    # exact in fp64 for the fp32-rounded f: compare with h^2 (f32 - f64) scale
    u = (ch * np.sin(math.pi * X) * np.sin(math.pi * Y)).reshape(-1)
    res = o.residual(u)
    assert np.max(np.abs(res)) < 4 * h * h * 2 * math.pi ** 2 * 2 ** -24
    # the sign reading: -div(grad p) = f  ->  p = +sin sin (not -sin sin)
    assert np.max(np.abs(o.residual(-u))) > 1e-3


def test_P4_residual_zero_polynomial():
    """u = x(1-x)y(1-y), f = 2[x(1-x)+y(1-y)]: the 5-point stencil is exact on quadratics."""
    N = 16
    h = 1.0 / N
    X, Y = W.grid_xy(N)
    f = (2 * (X * (1 - X) + Y * (1 - Y))).astype(np.float32)
    o = _ctx(N, f=f.reshape(-1))
    u = (X * (1 - X) * Y * (1 - Y)).reshape(-1)
    assert np.max(np.abs(o.residual(u))) < 8 * h * h * 2 ** -24


def test_P4_direct_solve_variable_alpha_gives_zero_loss():
    """u* = dense solve of the assembled discrete system (variable alpha) -> LOSS <= 1e-18."""
    N = 12
    K, S, f = W.random_fields(N, seed=11)
    o = _ctx(N, K=K, S=S, f=f)
    n, nn = N - 1, (N + 1) ** 2
    interior = [(j * (N + 1) + i) for j in range(1, N) for i in range(1, N)]
    # assemble the discrete operator from the brute-force literal Eq. 25 (P3's reference)
    alpha = o.alpha()
    zero_f = np.zeros(nn)
    cols = []
    for p in interior:
        e = np.zeros(nn)
        e[p] = 1.0
        cols.append(_literal_residual(N, alpha, e, zero_f))
    A = np.column_stack(cols)
    b = (f.astype(np.float64).reshape(N + 1, N + 1)[1:-1, 1:-1] / N ** 2).reshape(-1)
    ustar = np.zeros(nn)
    ustar[interior] = np.linalg.solve(A, b)
    loss, res, _ = o.loss_u(ustar)
    assert np.max(np.abs(res)) < 1e-12 and loss <= 1e-18


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 2.0])
def test_P5_loss_closed_form(beta):
    """alpha=1, f=2 pi^2 sin sin: LOSS(beta sin sin) = 2 sin^2(pi h/2) (c_h - beta)^2 [derived]."""
    N = 32
    h = 1.0 / N
    X, Y = W.grid_xy(N)
    f = (2 * math.pi ** 2 * np.sin(math.pi * X) * np.sin(math.pi * Y)).astype(np.float32)
    o = _ctx(N, f=f.reshape(-1))
    ch = (math.pi * h / 2) ** 2 / math.sin(math.pi * h / 2) ** 2
    want = 2 * math.sin(math.pi * h / 2) ** 2 * (ch - beta) ** 2
    loss, _, _ = o.loss_u((beta * np.sin(math.pi * X) * np.sin(math.pi * Y)).reshape(-1))
    assert abs(loss - want) <= 1e-6 * max(want, 1e-3)
    if beta == 0.0:
        assert abs(loss - 4.823015329536e-3) < 1e-8


# --------------------------------------------------------------------------- P6: inf-sup bounds
def test_P6_robust_loss_bounds():
    """gamma^2 h^2 e^T T e <= LOSS <= C^2 h^2 e^T T e, e = u - u*, gamma/C = min/max alpha."""
    N = 10
    K, S, f = W.random_fields(N, seed=5, kmin=0.3, kmax=3.0)
    o = _ctx(N, K=K, S=S, f=f)
    nn, n = (N + 1) ** 2, N - 1
    interior = [(j * (N + 1) + i) for j in range(1, N) for i in range(1, N)]
    A = np.column_stack([o.residual(np.eye(nn)[:, p]) - o.residual(np.zeros(nn)) for p in interior])
    b = -o.residual(np.zeros(nn))
    ustar = np.zeros(nn)
    ustar[interior] = np.linalg.solve(A, b)
    used = o.alpha().reshape(N + 1, N + 1)[:N, :N]     # nodes whose grad+ enters Eq. 25
    gamma, C = used.min(), used.max()
    T1 = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    T = np.kron(np.eye(n), T1) + np.kron(T1, np.eye(n))
    rng = np.random.default_rng(2)
    for _ in range(5):
        u = ustar.copy()
        u[interior] += rng.standard_normal(n * n)
        e = (u - ustar)[interior]
        loss, _, _ = o.loss_u(u)
        eTe = e @ T @ e / N ** 2
        assert gamma ** 2 * eTe * (1 - 1e-10) <= loss <= C ** 2 * eTe * (1 + 1e-10)


# --------------------------------------------------------------------------- P7: adjoint
def test_P7_adjoint_and_symmetry():
    """<A u, w> = <u, A^T w>; A symmetric; alpha=1: g_u = 2 h^2 RES [derived]."""
    N = 9
    K, S, f = W.random_fields(N, seed=9)
    o = _ctx(N, K=K, S=S, f=f)
    nn, n = (N + 1) ** 2, N - 1
    rng = np.random.default_rng(4)
    mask = np.zeros((N + 1, N + 1))
    mask[1:-1, 1:-1] = 1
    mask = mask.reshape(-1)
    r0 = o.residual(np.zeros(nn))
    u = rng.standard_normal(nn) * mask
    v = rng.standard_normal(nn) * mask
    w = rng.standard_normal(n * n)
    Au = o.residual(u) - r0
    Av = o.residual(v) - r0
    assert abs(Au @ w - u @ o.residual_adjoint(w)) < 1e-12 * np.abs(Au).sum() * np.abs(w).max()
    def interior(x):
        return x.reshape(N + 1, N + 1)[1:-1, 1:-1].reshape(-1)
    assert abs(Au @ interior(v) - Av @ interior(u)) < 1e-12 * (np.abs(Au).sum() + np.abs(Av).sum())
    # alpha = 1: the Gram cancels
    X, Y = W.grid_xy(N)
    o1 = _ctx(N, f=f, theta=W.random_theta((2, 8, 1), 1))
    loss, g, it = o1.loss_grad(intermediates=True)
    np.testing.assert_allclose(interior(it["gu"]), 2 * it["res"] / N ** 2, rtol=1e-10, atol=1e-16)


# --------------------------------------------------------------------------- P8: gradient vs FD
@pytest.mark.parametrize("widths,N,seed", [((2, 8, 1), 8, 0), ((2, 16, 16, 1), 8, 1),
                                           ((2, 32, 32, 1), 10, 2), ((2, 64, 64, 64, 1), 8, 3)])
def test_P8_gradient_vs_central_fd(widths, N, seed):
    K, S, f = W.random_fields(N, seed=seed)
    th = W.random_theta(widths, seed).astype(np.float64)
    o = _ctx(N, widths, K, S, f, th)
    loss, g = o.loss_grad(th)
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(th), size=min(len(th), 40), replace=False)
    for k in idx:
        step = 1e-6 * max(1.0, abs(th[k]))
        tp, tm = th.copy(), th.copy()
        tp[k] += step
        tm[k] -= step
        fd = (o.loss_grad(tp)[0] - o.loss_grad(tm)[0]) / (2 * step)
        assert abs(fd - g[k]) <= 1e-6 * max(abs(g[k]), 1e-3 * np.abs(g).max()), (k, fd, g[k])


# --------------------------------------------------------------------------- P9: Adam
def test_P9_adam_first_step_closed_form():
    """Step 1: m_hat = g, v_hat = g^2  ->  theta_1 = theta_0 - lr g/(|g| + eps)."""
    N = 8
    K, S, f = W.random_fields(N, seed=2)
    th0 = W.random_theta((2, 8, 1), 2)
    o = _ctx(N, (2, 8, 1), K, S, f, th0, lr=1e-2)
    _, g = o.loss_grad()
    o.adam_step(g)
    want = th0.astype(np.float64) - 1e-2 * g / (np.abs(g) + 1e-8)
    np.testing.assert_allclose(o.theta, want, rtol=1e-14, atol=1e-16)


def test_P9_adam_vs_torch_optim():
    torch = pytest.importorskip("torch")
    N = 8
    K, S, f = W.random_fields(N, seed=3)
    th0 = W.random_theta((2, 16, 16, 1), 3)
    o = _ctx(N, (2, 16, 16, 1), K, S, f, th0, lr=3e-3)
    p = torch.nn.Parameter(torch.tensor(th0.astype(np.float64)))
    opt = torch.optim.Adam([p], lr=3e-3, betas=(0.9, 0.999), eps=1e-8)
    for _ in range(10):
        _, g = o.loss_grad(p.detach().numpy())
        p.grad = torch.tensor(g)
        opt.step()
        o.adam_step(g)
    np.testing.assert_allclose(o.theta, p.detach().numpy(), rtol=1e-13, atol=1e-15)


# --------------------------------------------------------------------------- P10: torch autograd
def _torch_loss(torch, N, widths, theta, alpha, f):
    """Independent implementation: torch MLP + shifted-slice stencil + eigenbasis Gram inverse."""
    h = 1.0 / N
    n = N - 1
    th = theta
    c = torch.arange(N + 1, dtype=torch.float64) / N
    Y, X = torch.meshgrid(c, c, indexing="ij")
    z = torch.stack([X[1:-1, 1:-1].reshape(-1), Y[1:-1, 1:-1].reshape(-1)], 1)
    off = 0
    a = z
    for l in range(len(widths) - 1):
        fin, fout = widths[l], widths[l + 1]
        Wm = th[off:off + fin * fout].reshape(fout, fin)
        off += fin * fout
        bb = th[off:off + fout]
        off += fout
        a = a @ Wm.T + bb
        if l < len(widths) - 2:
            a = torch.tanh(a)
    cut = 16 * X * (1 - X) * Y * (1 - Y)
    U = torch.zeros(N + 1, N + 1, dtype=torch.float64)
    U = U.index_put((torch.arange(1, N).repeat_interleave(n), torch.arange(1, N).repeat(n)),
                    a[:, 0] * cut[1:-1, 1:-1].reshape(-1))
    A = torch.tensor(alpha.reshape(N + 1, N + 1))
    c0 = U[1:-1, 1:-1]
    res = (A[1:-1, 0:-2] * (c0 - U[1:-1, 0:-2]) + A[0:-2, 1:-1] * (c0 - U[0:-2, 1:-1])
           + A[1:-1, 1:-1] * (c0 - U[1:-1, 2:]) + A[1:-1, 1:-1] * (c0 - U[2:, 1:-1])
           - h * h * torch.tensor(f.reshape(N + 1, N + 1)[1:-1, 1:-1].astype(np.float64)))
    S, lam = _dst_matrix(N)
    S = torch.tensor(S)
    lam = torch.tensor(lam)
    Z = (S @ res @ S) / (lam[:, None] + lam[None, :])
    q = h * h * (S @ Z @ S)
    return (res * q).sum()


@pytest.mark.parametrize("name,Nred", [("C1", None), ("C2", None), ("C3", 32), ("C4", 16), ("C5", 16)])
def test_P10_loss_grad_vs_torch_autograd(name, Nred):
    torch = pytest.importorskip("torch")
    F = W.make_fields(name)
    w = F.workload
    N = w.N if Nred is None else Nred
    if Nred is None:
        K, S, f = F.K, F.S, F.f
    else:
        K, S, f = W.random_fields(N, seed=w.N)
    th = W.random_theta(w.widths, 7).astype(np.float64)
    o = _ctx(N, w.widths, K, S, f, th)
    loss, g = o.loss_grad()
    p = torch.tensor(th, requires_grad=True)
    tl = _torch_loss(torch, N, w.widths, p, o.alpha(), f)
    tl.backward()
    assert abs(loss - tl.item()) <= 1e-10 * abs(tl.item())
    np.testing.assert_allclose(g, p.grad.numpy(), rtol=1e-8, atol=1e-10 * np.abs(g).max())


# --------------------------------------------------------------------------- P11: convergence
def test_P11_training_converges_to_closed_form():
    """C1 (BASELINE.json configs[0]): 2000 Adam steps, lr 1e-3 -> rel-L2(u, c_h sin sin) <= 1e-2."""
    F = W.make_fields("C1")
    w = F.workload
    o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    hist = o.train(2000)
    N = w.N
    h = 1.0 / N
    X, Y = W.grid_xy(N)
    ch = (math.pi * h / 2) ** 2 / math.sin(math.pi * h / 2) ** 2
    ustar = (ch * np.sin(math.pi * X) * np.sin(math.pi * Y)).reshape(-1)
    u = o.forward()
    assert np.linalg.norm(u - ustar) / np.linalg.norm(ustar) <= 1e-2
    assert hist[-1] < 1e-2 * hist[0]   # SPEC.md:441 asks >= 1000x for its own init; see DESIGN.md


# --------------------------------------------------------------------------- P12, P13
def test_P12_cutoff_boundary_exact_zero():
    N = 16
    o = _ctx(N, (2, 8, 8, 1), theta=W.random_theta((2, 8, 8, 1), 0))
    U = o.forward().reshape(N + 1, N + 1)
    assert np.all(U[0, :] == 0) and np.all(U[-1, :] == 0) and np.all(U[:, 0] == 0) and np.all(U[:, -1] == 0)
    assert np.count_nonzero(U[1:-1, 1:-1]) == (N - 1) ** 2


def test_P12_cutoff_normalisation():
    """cutoff(1/2,1/2) = 1: a net that outputs the constant 1 gives u(1/2,1/2) = 1."""
    N = 8
    widths = (2, 4, 1)
    th = np.zeros(2 * 4 + 4 + 4 * 1 + 1)
    th[-1] = 1.0      # output bias
    o = _ctx(N, widths, theta=th.astype(np.float32))
    U = o.forward().reshape(N + 1, N + 1)
    assert U[N // 2, N // 2] == 1.0


def test_P13_zero_output_layer():
    """Zero output layer => u = 0, RES = -b, LOSS = b^T G^-1 b."""
    N = 16
    K, S, f = W.random_fields(N, seed=13)
    widths = (2, 16, 1)
    th = W.random_theta(widths, 13)
    th[-(16 + 1):] = 0.0
    o = _ctx(N, widths, K, S, f, th)
    loss, g, it = o.loss_grad(intermediates=True)
    assert np.all(it["u"] == 0.0)
    b = f.astype(np.float64).reshape(N + 1, N + 1)[1:-1, 1:-1].reshape(-1) / N ** 2
    np.testing.assert_allclose(it["res"], -b, rtol=1e-15)
    assert abs(loss - b @ _gram_inv_dst(N, b)) <= 1e-11 * loss


# --------------------------------------------------------------------------- P14: gravity term (f1)
# Eq. 23's RHS carries grad+ . (g K ((1-S) rho_w/mu_w + S rho_g/mu_g)); reading R23
# makes it non-dimensional: F = (0, -Gr) K ((1-S) + M r S), r = rho_g/rho_w, and b = h^2 (f - grad+.F).
def _gamma(K, S, r=oracle.DENSITY_RATIO):
    s = np.clip(S.astype(np.float64), 0.0, 1.0)
    return K.astype(np.float64) * ((1.0 - s) + oracle.MOBILITY_RATIO * r * s)


def test_P14_gravity_vanishes_for_homogeneous_medium():
    """Constant K and S: F is constant, its forward-difference divergence is exactly 0."""
    N = 16
    nn = (N + 1) ** 2
    K = np.full(nn, 2.5, np.float32)
    S = np.full(nn, 0.25, np.float32)
    f = W.random_fields(N, seed=3)[2]
    b0 = _ctx(N, K=K, S=S, f=f).rhs()
    b1 = _ctx(N, K=K, S=S, f=f, gravity=1.7).rhs()
    assert np.array_equal(b0, b1)


def test_P14_gravity_linear_permeability_is_a_constant_source():
    """K = 1 + c y, S = 0: gamma_{k,l+1} - gamma_{k,l} = c h, so b(Gr) - b(0) = h^2 Gr c exactly on
    every node with l < N; and the loss equals the gravity-free problem with f + Gr c."""
    N, c, Gr = 16, 0.5, 0.75
    j = np.repeat(np.arange(N + 1), N + 1)
    K = (1.0 + c * j / N).astype(np.float32)        # exact in fp32
    f = W.random_fields(N, seed=4)[2]
    widths = (2, 8, 8, 1)
    th = W.random_theta(widths, 4)
    og = _ctx(N, widths, K=K, f=f, theta=th, gravity=Gr)
    o0 = _ctx(N, widths, K=K, f=(f.astype(np.float64) + Gr * c).astype(np.float32), theta=th)
    d = (og.rhs() - _ctx(N, widths, K=K, f=f, theta=th).rhs()).reshape(N + 1, N + 1)
    np.testing.assert_allclose(d[:N, :N], Gr * c / N ** 2, rtol=1e-12)   # grad+ needs (i+1, j), (i, j+1)
    assert abs(og.loss_grad()[0] - o0.loss_grad()[0]) <= 1e-6 * o0.loss_grad()[0]


def test_P14_gravity_column_sums_telescope():
    """sum over l = 1..N-1 of the gravity part of b at column k = h Gr (gamma_{k,N} - gamma_{k,1}):
    catches a wrong sign, difference direction (forward vs backward) or power of h."""
    N, Gr = 32, -1.3
    K, S, f = W.random_fields(N, seed=5)
    d = (_ctx(N, K=K, S=S, f=f, gravity=Gr).rhs() - _ctx(N, K=K, S=S, f=f).rhs()).reshape(N + 1, N + 1)
    g = _gamma(K, S).reshape(N + 1, N + 1)
    lhs = d[1:N, :].sum(axis=0)                      # rows = l (y), columns = k (x)
    rhs = Gr / N * (g[N, :] - g[1, :])
    np.testing.assert_allclose(lhs[1:N], rhs[1:N], rtol=1e-10, atol=1e-14)


def test_P14_gravity_saturation_dependence_and_update():
    """K = 1 and S = y/2: gamma steps by (M r - 1) h / 2 per row, so b(Gr) - b(0) = h^2 Gr (M r - 1)/2;
    set_saturation must recompute it (the term depends on S through rho_g/rho_w)."""
    N, Gr = 16, 0.9
    nn = (N + 1) ** 2
    j = np.repeat(np.arange(N + 1), N + 1)
    S_lin = (0.5 * j / N).astype(np.float32)
    o = _ctx(N, gravity=Gr)
    b_S0 = o.rhs().copy()
    o.set_saturation(S_lin)
    d = (o.rhs() - b_S0).reshape(N + 1, N + 1)
    expect = Gr * (oracle.MOBILITY_RATIO * oracle.DENSITY_RATIO - 1.0) / 2.0 / N ** 2
    np.testing.assert_allclose(d[:N, :N], expect, rtol=1e-12)
    assert np.all(d[N, :] == 0.0) and np.all(d[:, N] == 0.0)
    assert np.allclose(_ctx(N, S=S_lin, gravity=Gr).rhs(), o.rhs(), rtol=0, atol=1e-15)
    del nn


# --------------------------------------------------------------------------- P15: continuous evaluation (f1)
def test_P15_eval_points_boundary_zero_and_lattice_consistency():
    N = 16
    widths = (2, 8, 8, 1)
    o = _ctx(N, widths, theta=W.random_theta(widths, 6))
    t = np.linspace(0.0, 1.0, 23)
    edge = np.concatenate([np.stack([np.zeros_like(t), t], 1), np.stack([np.ones_like(t), t], 1),
                           np.stack([t, np.zeros_like(t)], 1), np.stack([t, np.ones_like(t)], 1)])
    assert np.all(o.eval_points(edge) == 0.0)
    i, j = np.meshgrid(np.arange(N + 1), np.arange(N + 1))
    xy = np.stack([i.reshape(-1) / N, j.reshape(-1) / N], 1)
    np.testing.assert_array_equal(o.eval_points(xy), o.forward())


def test_P15_eval_points_closed_form_one_neuron():
    """widths (2, 1, 1): p(x,y) = 16x(1-x)y(1-y) (w2 tanh(a x + b y + c) + d), numpy's tanh."""
    a, b, c, w2, d = 0.7, -1.3, 0.2, 1.5, -0.4
    th = np.array([a, b, c, w2, d], np.float32)
    o = _ctx(8, (2, 1, 1), theta=th)
    rng = np.random.default_rng(7)
    xy = rng.uniform(-0.5, 1.5, size=(200, 2))      # outside the unit square too
    x, y = xy[:, 0], xy[:, 1]
    t64 = th.astype(np.float64)
    ref = 16 * x * (1 - x) * y * (1 - y) * (t64[3] * np.tanh(t64[0] * x + t64[1] * y + t64[2]) + t64[4])
    np.testing.assert_allclose(o.eval_points(xy), ref, rtol=1e-13, atol=1e-15)


# --------------------------------------------------------------------------- P16: direct solve (f2)
def test_P16_direct_solve_zero_residual_and_dense_lapack():
    """u* = A(alpha)^-1 b: RES(u*) = 0 by the literal residual (P3-pinned), LOSS(u*) = 0, and equal to a
    dense LAPACK solve of the matrix assembled column by column from orc_residual (N = 8)."""
    N = 8
    K, S, f = W.random_fields(N, seed=16)
    o = _ctx(N, K=K, S=S, f=f, gravity=0.6)
    u = o.direct_solve()
    U = u.reshape(N + 1, N + 1)
    assert np.all(U[0] == 0) and np.all(U[-1] == 0) and np.all(U[:, 0] == 0) and np.all(U[:, -1] == 0)
    res = o.residual(u)
    assert np.max(np.abs(res)) <= 1e-12 * np.abs(o.rhs()).max()
    n = N - 1
    b = -o.residual(np.zeros((N + 1) ** 2))          # RES(0) = -b on the interior
    A = np.empty((n * n, n * n))
    for c in range(n * n):
        e = np.zeros((N + 1) ** 2)
        e[(c // n + 1) * (N + 1) + (c % n + 1)] = 1.0
        A[:, c] = o.residual(e) + b                   # A e = RES(e) + b
    x = np.linalg.solve(A, b)
    np.testing.assert_allclose(U[1:-1, 1:-1].reshape(-1), x, rtol=1e-11, atol=1e-14)


def test_P16_direct_solve_manufactured_polynomial():
    """alpha = 1, f = 2[x(1-x) + y(1-y)]: the 5-point stencil is exact on quadratics, so u* = x(1-x)y(1-y)."""
    N = 32
    i, j = np.meshgrid(np.arange(N + 1), np.arange(N + 1))
    x, y = (i / N).reshape(-1), (j / N).reshape(-1)
    f = (2.0 * (x * (1 - x) + y * (1 - y))).astype(np.float32)
    u = _ctx(N, f=f).direct_solve()
    ustar = x * (1 - x) * y * (1 - y)
    # f is rounded to fp32 on input: the solution error is that rounding propagated (~1e-8 rel)
    np.testing.assert_allclose(u, ustar, rtol=0, atol=1e-8 * ustar.max())


# --------------------------------------------------------------------------- P17-P19: IGA-ADS saturation step (f3)
def test_P17_spline_space_basis_quadrature_mass():
    """B-splines of degree r (Eq. 11): partition of unity, the cardinal quadratic at an interior element
    midpoint (1/8, 3/4, 1/8 by hand), open-knot interpolation at x = 0; the Gauss rule integrates x^k
    exactly for k <= 2r + 1; the mass matrix (Eq. 14) sums to 1, has bandwidth r, and for degree-1 hats
    on 2 elements equals the hand integrals [[1/6, 1/12, 0], [1/12, 1/3, 1/12], [0, 1/12, 1/6]]."""
    rng = np.random.default_rng(17)
    for ne, r in [(5, 1), (8, 2), (7, 3)]:
        o = oracle.IgaOracle(ne, r)
        assert o.nb == ne + r
        for x in rng.uniform(0, 1, 200):
            i0, v, d = o.basis(x)
            assert 0 <= i0 <= o.nb - r - 1 and np.all(v >= -1e-15)
            assert abs(v.sum() - 1) <= 1e-13 and abs(d.sum()) <= 1e-10
        i0, v, _ = o.basis(0.0)
        assert i0 == 0 and v[0] == 1.0 and np.all(v[1:] == 0)
        gx, gw = o.gauss()
        for k in range(2 * r + 2):
            assert abs(np.sum(gw * gx ** k) - 1.0 / (k + 1)) <= 1e-14
        M = o.mass_1d()
        assert abs(M.sum() - 1.0) <= 1e-13
        i, k = np.indices(M.shape)
        assert np.all(M[np.abs(i - k) > r] == 0.0)
    _, v, d = oracle.IgaOracle(8, 2).basis(3.5 / 8)
    np.testing.assert_allclose(v, [0.125, 0.75, 0.125], atol=1e-15)
    np.testing.assert_allclose(oracle.IgaOracle(2, 1).mass_1d(),
                               [[1 / 6, 1 / 12, 0], [1 / 12, 1 / 3, 1 / 12], [0, 1 / 12, 1 / 6]], atol=1e-15)


def test_P18_kronecker_solve_and_projection():
    """M = M^x (x) M^y (Eq. 14): the directional solves equal a dense solve of np.kron(M, M); a
    constructed load M C0 M recovers C0; the L2 projection reproduces constants and x^2 + y^2 in the
    quadratic space, preserves the integral, and eval's gradient matches central differences."""
    rng = np.random.default_rng(18)
    o = oracle.IgaOracle(4, 2)
    M = o.mass_1d()
    L = rng.standard_normal((o.nb, o.nb))
    C = o.kron_solve(L)
    x = np.linalg.solve(np.kron(M, M), L.reshape(-1))
    np.testing.assert_allclose(C.reshape(-1), x, rtol=1e-10, atol=1e-10)
    C0 = rng.standard_normal((o.nb, o.nb))
    np.testing.assert_allclose(o.kron_solve(M @ C0 @ M), C0, atol=1e-9)
    o = oracle.IgaOracle(16, 2)
    q = o.quad_points()
    np.testing.assert_allclose(o.project(np.ones(len(q))), 1.0, atol=1e-12)
    f = q[:, 0] ** 2 + q[:, 1] ** 2
    C = o.project(f)
    pts = rng.uniform(0, 1, (100, 2))
    np.testing.assert_allclose(o.eval(C, pts), pts[:, 0] ** 2 + pts[:, 1] ** 2, atol=1e-12)
    g = np.sin(np.pi * q[:, 0]) * np.sin(np.pi * q[:, 1])
    Cg = o.project(g)
    m1 = o.mass_1d().sum(axis=0)                      # int B_k dx
    assert abs(m1 @ Cg @ m1 - 4 / np.pi ** 2) <= 1e-6  # = int f (projection tested with v = 1)
    val, grad = o.eval(Cg, pts, grad=True)
    e = 1e-6
    fdx = (o.eval(Cg, pts + [e, 0]) - o.eval(Cg, pts - [e, 0])) / (2 * e)
    fdy = (o.eval(Cg, pts + [0, e]) - o.eval(Cg, pts - [0, e])) / (2 * e)
    np.testing.assert_allclose(grad[:, 0], fdx, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(grad[:, 1], fdy, rtol=1e-5, atol=1e-7)


def _blob(o, cx=0.5, cy=0.4, w=0.1):
    q = o.quad_points()
    C = o.project(np.exp(-((q[:, 0] - cx) ** 2 + (q[:, 1] - cy) ** 2) / (2 * w * w)))
    C[0, :] = C[-1, :] = C[:, 0] = C[:, -1] = 0.0
    return C


def test_P19_saturation_step_identities_and_source():
    """Eq. 10: tau = 0, or grad p = 0 with no gravity and no source, is the identity on spline data
    with zero boundary coefficients; a pure source adds exactly the projection of (tau/phi) q."""
    o = oracle.IgaOracle(16, 2)
    S = _blob(o)
    ne = o.ne
    K = np.random.default_rng(19).uniform(0.5, 2.0, (ne, ne))
    P = np.random.default_rng(20).standard_normal((o.nb, o.nb))
    np.testing.assert_allclose(o.saturation_step(S, P, K, np.zeros((ne, ne)), tau=0.0, gravity=1.0), S, atol=1e-12)
    np.testing.assert_allclose(o.saturation_step(S, np.zeros_like(P), K, np.zeros((ne, ne)), tau=0.3), S, atol=1e-12)
    q = np.zeros((ne, ne))
    q[6:10, 6:10] = 2.0
    tau, phi = 0.05, 0.4
    d = o.saturation_step(np.zeros_like(S), np.zeros_like(P), K, q, tau=tau, phi=phi)
    qq = o.quad_points()
    qf = q[np.minimum((qq[:, 1] * ne).astype(int), ne - 1), np.minimum((qq[:, 0] * ne).astype(int), ne - 1)]
    ref = o.project(tau / phi * qf)
    ref[0, :] = ref[-1, :] = ref[:, 0] = ref[:, -1] = 0.0
    np.testing.assert_allclose(d, ref, atol=1e-12)


def test_P19_saturation_step_buoyancy_and_mass():
    """Hydrostatic water pressure p = -Gr y (grad p = rho_w g, R23 units) and K = 1: the gas flux is
    M S K Gr (1 - rho_g/rho_w) upward, so the blob's centroid rises (the sign that reading R24 fixes;
    Eq. 9 as printed would make it sink) while the gas mass is conserved (interior blob, q = 0)."""
    o = oracle.IgaOracle(32, 2)
    S = _blob(o, cy=0.4)
    q = o.quad_points()
    Gr = 2.0
    P = o.project(-Gr * q[:, 1])
    ne = o.ne
    S1 = o.saturation_step(S, P, np.ones((ne, ne)), np.zeros((ne, ne)), tau=2e-3, gravity=Gr)
    g = np.stack(np.meshgrid(np.linspace(0, 1, 201), np.linspace(0, 1, 201)), -1).reshape(-1, 2)
    s0, s1 = o.eval(S, g), o.eval(S1, g)
    cy0, cy1 = (s0 * g[:, 1]).sum() / s0.sum(), (s1 * g[:, 1]).sum() / s1.sum()
    assert cy1 > cy0 + 1e-4, (cy0, cy1)
    m1 = o.mass_1d().sum(axis=0)
    assert abs(m1 @ S1 @ m1 - m1 @ S @ m1) <= 1e-4 * (m1 @ S @ m1)   # blob tails reach the zeroed boundary


# ------------------------------------------------------------------ P21: the 11-bit precision-class model
def test_P21_round_sig_is_11_bit_round_to_nearest():
    """round_sig keeps 11 significant bits with round-to-nearest-even at any magnitude: exact on
    11-bit values, relative error <= 2^-11 otherwise, ties to even, sign symmetric, idempotent."""
    from oracle.precision_model import round_sig
    rng = np.random.default_rng(3)
    for scale in (1e-9, 1e-3, 1.0, 1e4, 1e9):
        a = rng.standard_normal(4096) * scale
        r = round_sig(a)
        assert np.all(np.abs(r - a) <= 2.0 ** -11 * np.abs(a) * (1 + 1e-12))
        np.testing.assert_array_equal(round_sig(r), r)
        np.testing.assert_array_equal(round_sig(-a), -r)
    m = np.ldexp(np.arange(1024, 2048, dtype=np.float64), -10)     # all 11-bit significands in [1, 2)
    np.testing.assert_array_equal(round_sig(m), m)
    x = np.array([2.0, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11])        # ties between 11-bit neighbours
    np.testing.assert_array_equal(round_sig(x), [2.0, 1.0, 1.0 + 4 * 2.0 ** -11])


def test_P21_precision_model_unrounded_is_the_oracle():
    """With no rounding the model's iteration is the oracle's (its forward and backward are a second,
    numpy implementation of PAPER.md:373 and the chain rule): gradient to 1e-12, 5-step history."""
    from oracle.precision_model import PrecisionModel
    N, widths = 16, (2, 32, 32, 32, 1)
    K, S, f = W.random_fields(N, 17)
    th = W.random_theta(widths, 17)
    pm = PrecisionModel(N, widths, K, S, f, th, bits=None)
    o = oracle.Oracle(N, widths, K, S, f, th)
    l, g = pm.loss_grad()
    rl, rg = o.loss_grad()
    assert abs(l - rl) <= 1e-13 * abs(rl)
    assert np.linalg.norm(g - rg) <= 1e-12 * np.linalg.norm(rg)
    np.testing.assert_allclose(pm.train(5), o.train(5), rtol=1e-11)
    pm11 = PrecisionModel(N, widths, K, S, f, th, bits=11)
    l11, g11 = pm11.loss_grad()
    assert l11 == l                                        # the forward is not rounded
    assert 0 < np.linalg.norm(g11 - rg) <= 1e-2 * np.linalg.norm(rg)


def test_oracle_state_resume_is_exact():
    """scripts/oracle_runs.py resumes long fixture runs (C5's schedule) from the saved fp64 state:
    theta + Adam (m, v, t) restored into a fresh oracle continue the iteration bit for bit."""
    N, widths = 16, (2, 32, 32, 1)
    K, S, f = W.random_fields(N, 71)
    th = W.random_theta(widths, 71)
    a = oracle.Oracle(N, widths, K, S, f, th)
    full = a.train(6)
    b = oracle.Oracle(N, widths, K, S, f, th)
    first = b.train(3)
    m, v, t = b.adam_state()
    c = oracle.Oracle(N, widths, K, S, f, th)
    c.theta = b.theta
    c.set_adam_state(m, v, t)
    rest = c.train(3)
    np.testing.assert_array_equal(np.concatenate([first, rest]), full)
    np.testing.assert_array_equal(c.theta, a.theta)
    assert c.adam_state()[2] == 6
