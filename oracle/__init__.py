"""ctypes wrapper of the fp64 CPU oracle (oracle/crvpinn_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg. The product package never imports it.

Every function follows the paper step by step; see the header of crvpinn_oracle.c for the
passage each step cites and DESIGN.md §4 for the pins (P1..P13) in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "crvpinn_oracle.c")
_SRC_IGA = os.path.join(_HERE, "iga_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_SRC_ABI = os.path.join(_HERE, "crvpinn_abi.c")
LIB_ABI = os.path.join(_HERE, "liboracle_abi.so")   # the oracle behind the product's C ABI (tests only)

MOBILITY_RATIO = 25.35 / 3.95   # Table 1
DENSITY_RATIO = 479.0 / 1045.0   # rho_g / rho_w, Table 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, OpenMP)."""
    if (force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC)
            or os.path.getmtime(_LIB) < os.path.getmtime(_SRC_IGA)):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC, _SRC_IGA, "-lm"])
    if (force or not os.path.exists(LIB_ABI) or os.path.getmtime(LIB_ABI) < os.path.getmtime(_SRC)
            or os.path.getmtime(LIB_ABI) < os.path.getmtime(_SRC_ABI)):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-fvisibility=default", "-o", LIB_ABI,
                               _SRC, _SRC_ABI, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        D = ctypes.POINTER(ctypes.c_double)
        F = ctypes.POINTER(ctypes.c_float)
        I = ctypes.POINTER(ctypes.c_int)
        L.orc_create.restype = P
        L.orc_create.argtypes = [ctypes.c_int, ctypes.c_int, I, F, F, F, F, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.orc_destroy.argtypes = [P]
        L.orc_num_params.restype = ctypes.c_long
        L.orc_num_params.argtypes = [P]
        L.orc_get_theta.argtypes = [P, D]
        L.orc_set_theta.argtypes = [P, D]
        L.orc_get_adam.argtypes = [P, D, D, ctypes.POINTER(ctypes.c_long)]
        L.orc_set_adam.argtypes = [P, D, D, ctypes.c_long]
        L.orc_get_alpha.argtypes = [P, D]
        L.orc_get_b.argtypes = [P, D]
        L.orc_direct_solve.restype = ctypes.c_int
        L.orc_direct_solve.argtypes = [P, D]
        L.orc_eval_points.argtypes = [P, D, ctypes.c_long, D, D]
        L.orc_set_saturation.argtypes = [P, F, F]
        L.orc_forward.argtypes = [P, D, D]
        L.orc_forward_rows.argtypes = [P, D, ctypes.c_int, ctypes.c_int, D]
        L.orc_grad_rows.argtypes = [P, D, D, ctypes.c_int, ctypes.c_int, D]
        L.orc_residual.argtypes = [P, D, D]
        L.orc_residual_adjoint.argtypes = [P, D, D]
        L.orc_gram_solve.argtypes = [P, D, D]
        L.orc_gram_matvec.argtypes = [P, D, D]
        L.orc_loss_u.restype = ctypes.c_double
        L.orc_loss_u.argtypes = [P, D, D, D]
        L.orc_loss_grad.restype = ctypes.c_double
        L.orc_loss_grad.argtypes = [P, D, D, D, D, D, D]
        L.orc_adam_step.argtypes = [P, D]
        L.orc_train.restype = ctypes.c_int
        L.orc_train.argtypes = [P, ctypes.c_int, D]
        L.orc_max_threads.restype = ctypes.c_int
        # IGA-ADS saturation step (iga_oracle.c)
        L.iga_create.restype = P
        L.iga_create.argtypes = [ctypes.c_int, ctypes.c_int]
        L.iga_destroy.argtypes = [P]
        L.iga_num_basis.restype = ctypes.c_int
        L.iga_num_basis.argtypes = [P]
        L.iga_mass_1d.argtypes = [P, D]
        L.iga_gauss.argtypes = [P, D, D]
        L.iga_basis.restype = ctypes.c_int
        L.iga_basis.argtypes = [P, ctypes.c_double, D, D]
        L.iga_quad_points.argtypes = [P, D]
        L.iga_kron_solve.argtypes = [P, D, D]
        L.iga_load.argtypes = [P, D, D]
        L.iga_project.argtypes = [P, D, D]
        L.iga_eval.argtypes = [P, D, ctypes.c_long, D, D, D]
        L.iga_saturation_step.argtypes = [P, D, D, D, D, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_double, D]
        _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


class Oracle:
    """One CRVPINN problem: grid N, widths, inputs K, S, f, parameters and Adam state."""

    def __init__(self, N: int, widths, K, S, f, theta0=None, *, mobility: float = MOBILITY_RATIO,
                 lr: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 factor_gram: bool = True, gravity: float = 0.0, density_ratio: float = DENSITY_RATIO):
        L = lib()
        self.N, self.n = int(N), int(N) - 1
        self.widths = tuple(int(w) for w in widths)
        w = (ctypes.c_int * len(self.widths))(*self.widths)
        self._K, self._S, self._f = _f32(K), _f32(S), _f32(f)
        th = None if theta0 is None else _f32(theta0)
        self._h = L.orc_create(self.N, len(self.widths) - 1, w, _fp(self._K), _fp(self._S),
                               _fp(self._f), None if th is None else _fp(th), mobility, lr,
                               beta1, beta2, eps, 1 if factor_gram else 0, gravity, density_ratio)
        if not self._h:
            raise MemoryError("orc_create failed")
        self.np = int(L.orc_num_params(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    # -- state
    @property
    def theta(self) -> np.ndarray:
        out = np.empty(self.np)
        lib().orc_get_theta(self._h, _dp(out))
        return out

    @theta.setter
    def theta(self, th):
        th = np.ascontiguousarray(th, dtype=np.float64)
        lib().orc_set_theta(self._h, _dp(th))

    def adam_state(self):
        m, v, t = np.empty(self.np), np.empty(self.np), ctypes.c_long(0)
        lib().orc_get_adam(self._h, _dp(m), _dp(v), ctypes.byref(t))
        return m, v, int(t.value)

    def set_adam_state(self, m, v, t: int):
        m = np.ascontiguousarray(m, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        lib().orc_set_adam(self._h, _dp(m), _dp(v), int(t))

    def alpha(self) -> np.ndarray:
        out = np.empty((self.N + 1) ** 2)
        lib().orc_get_alpha(self._h, _dp(out))
        return out

    def rhs(self) -> np.ndarray:
        """b = h^2 (f - grad+ . F) on the (N+1)^2 lattice (A0 with the gravity term)."""
        out = np.empty((self.N + 1) ** 2)
        lib().orc_get_b(self._h, _dp(out))
        return out

    def direct_solve(self) -> np.ndarray:
        """u* with A(alpha) u* = b (band LU, fp64), (N+1)^2 lattice."""
        out = np.empty((self.N + 1) ** 2)
        if lib().orc_direct_solve(self._h, _dp(out)) != 0:
            raise MemoryError("orc_direct_solve: allocation failed")
        return out

    def eval_points(self, xy, theta=None) -> np.ndarray:
        """cutoff(x, y) * net(x, y) at arbitrary points xy (n, 2), fp64."""
        th = self.theta if theta is None else np.ascontiguousarray(theta, dtype=np.float64)
        xy = np.ascontiguousarray(np.asarray(xy, dtype=np.float64).reshape(-1, 2))
        out = np.empty(xy.shape[0])
        lib().orc_eval_points(self._h, _dp(th), int(xy.shape[0]), _dp(xy), _dp(out))
        return out

    def set_saturation(self, S, K=None):
        self._S = _f32(S)
        if K is not None:
            self._K = _f32(K)
        lib().orc_set_saturation(self._h, _fp(self._K), _fp(self._S))

    # -- steps
    def forward(self, theta=None) -> np.ndarray:
        th = self.theta if theta is None else np.ascontiguousarray(theta, dtype=np.float64)
        u = np.empty((self.N + 1) ** 2)
        lib().orc_forward(self._h, _dp(th), _dp(u))
        return u

    def forward_rows(self, j0: int, j1: int, theta=None) -> np.ndarray:
        """u at the interior nodes of rows j in [j0, j1), zero elsewhere (one shard's forward)."""
        th = self.theta if theta is None else np.ascontiguousarray(theta, dtype=np.float64)
        u = np.empty((self.N + 1) ** 2)
        lib().orc_forward_rows(self._h, _dp(th), int(j0), int(j1), _dp(u))
        return u

    def grad_rows(self, gu, j0: int, j1: int, theta=None) -> np.ndarray:
        """dLOSS/dtheta over the MLP points of rows [j0, j1), given gu = dLOSS/du (one shard's backward)."""
        th = self.theta if theta is None else np.ascontiguousarray(theta, dtype=np.float64)
        gu = np.ascontiguousarray(gu, dtype=np.float64)
        g = np.empty(self.np)
        lib().orc_grad_rows(self._h, _dp(th), _dp(gu), int(j0), int(j1), _dp(g))
        return g

    def residual(self, u) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        r = np.empty(self.n * self.n)
        lib().orc_residual(self._h, _dp(u), _dp(r))
        return r

    def residual_adjoint(self, w) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64)
        g = np.empty((self.N + 1) ** 2)
        lib().orc_residual_adjoint(self._h, _dp(w), _dp(g))
        return g

    def gram_solve(self, rhs) -> np.ndarray:
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        q = np.empty(self.n * self.n)
        lib().orc_gram_solve(self._h, _dp(rhs), _dp(q))
        return q

    def gram_matvec(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty(self.n * self.n)
        lib().orc_gram_matvec(self._h, _dp(v), _dp(out))
        return out

    def loss_u(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        r, q = np.empty(self.n * self.n), np.empty(self.n * self.n)
        loss = lib().orc_loss_u(self._h, _dp(u), _dp(r), _dp(q))
        return loss, r, q

    def loss_grad(self, theta=None, intermediates: bool = False):
        th = None if theta is None else np.ascontiguousarray(theta, dtype=np.float64)
        g = np.empty(self.np)
        nn, n2 = (self.N + 1) ** 2, self.n * self.n
        if intermediates:
            u, r, q, gu = np.empty(nn), np.empty(n2), np.empty(n2), np.empty(nn)
            loss = lib().orc_loss_grad(self._h, None if th is None else _dp(th), _dp(g),
                                       _dp(u), _dp(r), _dp(q), _dp(gu))
            return loss, g, dict(u=u, res=r, q=q, gu=gu)
        loss = lib().orc_loss_grad(self._h, None if th is None else _dp(th), _dp(g),
                                   None, None, None, None)
        return loss, g

    def adam_step(self, grad):
        grad = np.ascontiguousarray(grad, dtype=np.float64)
        lib().orc_adam_step(self._h, _dp(grad))

    def train(self, n_iters: int) -> np.ndarray:
        hist = np.empty(n_iters)
        rc = lib().orc_train(self._h, int(n_iters), _dp(hist))
        if rc != 0:
            raise FloatingPointError("oracle loss became non-finite")
        return hist


def max_threads() -> int:
    return int(lib().orc_max_threads())


class IgaOracle:
    """Tensor-product B-spline space of degree r on [0,1]^2 with ne elements per axis (iga_oracle.c):
    the IGA-ADS saturation step of SURVEY.md §8(f) f3, fp64. Coefficient matrices are [l][k]
    (row = y basis index, column = x basis index), nb = ne + r per axis."""

    def __init__(self, ne: int, degree: int = 2):
        self.ne, self.r = int(ne), int(degree)
        self._h = lib().iga_create(self.ne, self.r)
        if not self._h:
            raise ValueError("iga_create: need ne >= 1 and 1 <= degree <= 8")
        self.nb = int(lib().iga_num_basis(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().iga_destroy(self._h)
            self._h = None

    def mass_1d(self) -> np.ndarray:
        out = np.empty((self.nb, self.nb))
        lib().iga_mass_1d(self._h, _dp(out))
        return out

    def gauss(self):
        x, w = np.empty(self.r + 1), np.empty(self.r + 1)
        lib().iga_gauss(self._h, _dp(x), _dp(w))
        return x, w

    def basis(self, x: float):
        val, der = np.empty(self.r + 1), np.empty(self.r + 1)
        i0 = lib().iga_basis(self._h, float(x), _dp(val), _dp(der))
        return int(i0), val, der

    def quad_points(self) -> np.ndarray:
        m = self.ne * (self.r + 1)
        out = np.empty((m * m, 2))
        lib().iga_quad_points(self._h, _dp(out))
        return out

    def kron_solve(self, L) -> np.ndarray:
        L = np.ascontiguousarray(L, dtype=np.float64).reshape(self.nb, self.nb)
        out = np.empty_like(L)
        lib().iga_kron_solve(self._h, _dp(L), _dp(out))
        return out

    def load(self, fq) -> np.ndarray:
        fq = np.ascontiguousarray(fq, dtype=np.float64).reshape(-1)
        out = np.empty((self.nb, self.nb))
        lib().iga_load(self._h, _dp(fq), _dp(out))
        return out

    def project(self, fq) -> np.ndarray:
        fq = np.ascontiguousarray(fq, dtype=np.float64).reshape(-1)
        out = np.empty((self.nb, self.nb))
        lib().iga_project(self._h, _dp(fq), _dp(out))
        return out

    def eval(self, C, xy, grad: bool = False):
        C = np.ascontiguousarray(C, dtype=np.float64).reshape(self.nb, self.nb)
        xy = np.ascontiguousarray(np.asarray(xy, dtype=np.float64).reshape(-1, 2))
        val = np.empty(xy.shape[0])
        g = np.empty((xy.shape[0], 2)) if grad else None
        lib().iga_eval(self._h, _dp(C), int(xy.shape[0]), _dp(xy), _dp(val), None if g is None else _dp(g))
        return (val, g) if grad else val

    def saturation_step(self, S, P, K, q, tau, phi=1.0, mobility=MOBILITY_RATIO, density_ratio=DENSITY_RATIO,
                        gravity=0.0) -> np.ndarray:
        S = np.ascontiguousarray(S, dtype=np.float64).reshape(self.nb, self.nb)
        P = np.ascontiguousarray(P, dtype=np.float64).reshape(self.nb, self.nb)
        K = np.ascontiguousarray(K, dtype=np.float64).reshape(self.ne, self.ne)
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(self.ne, self.ne)
        out = np.empty((self.nb, self.nb))
        lib().iga_saturation_step(self._h, _dp(S), _dp(P), _dp(K), _dp(q), float(tau), float(phi), float(mobility),
                                  float(density_ratio), float(gravity), _dp(out))
        return out
