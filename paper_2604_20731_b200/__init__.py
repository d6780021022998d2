"""Python binding of the CRVPINN sm_100a library (include/crvpinn.h).

Argument marshalling only: every step of the CRVPINN update runs in the CUDA kernels of
libcrvpinn.so. There is no CPU fallback: if the library is missing this module raises, and
without an sm_100 device every call fails with CRVPINN_ECUDA.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CRVPINN_LIB", os.path.join(_HERE, "libcrvpinn.so"))   # override: A/B builds

CRVPINN_OK, CRVPINN_EINVAL, CRVPINN_ENOMEM, CRVPINN_ECUDA, CRVPINN_ENONFINITE, CRVPINN_EDOMAIN = 0, -1, -2, -3, -4, -5
PREC_TENSOR, PREC_FP32 = 0, 1

# every symbol include/crvpinn.h declares
EXPORTS = [
    "crvpinn_default_opts", "crvpinn_create", "crvpinn_set_saturation", "crvpinn_set_saturation_device",
    "crvpinn_pretrain", "crvpinn_step", "crvpinn_eval", "crvpinn_eval_points", "crvpinn_direct_solve",
    "crvpinn_loss_grad",
    "crvpinn_get_intermediates",
    "crvpinn_num_params", "crvpinn_get_params", "crvpinn_set_params", "crvpinn_get_adam", "crvpinn_set_adam",
    "crvpinn_set_profiling", "crvpinn_get_profile", "crvpinn_launches_per_iter", "crvpinn_stream",
    "crvpinn_last_error", "crvpinn_destroy",
    "crvpinn_shard_tiles", "crvpinn_nccl_unique_id", "crvpinn_shard_forward", "crvpinn_shard_backward",
    "crvpinn_iga_create", "crvpinn_iga_num_basis", "crvpinn_iga_num_quad_points", "crvpinn_iga_quad_points",
    "crvpinn_iga_project", "crvpinn_iga_saturation_step", "crvpinn_iga_eval", "crvpinn_iga_last_ms",
    "crvpinn_iga_last_error", "crvpinn_iga_destroy",
]


class CrvpinnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"crvpinn error {code}: {msg}")
        self.code = code


class Opts(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("mobility_ratio", ctypes.c_double), ("precision", ctypes.c_int),
                ("seed", ctypes.c_uint64), ("stream", ctypes.c_void_p), ("device", ctypes.c_int),
                ("gravity", ctypes.c_double), ("density_ratio", ctypes.c_double),
                ("shard_rank", ctypes.c_int), ("shard_world", ctypes.c_int), ("nccl", ctypes.c_int),
                ("nccl_id", ctypes.c_ubyte * 128)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libcrvpinn.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2604_20731_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(path)
    P, F, D, I = ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double), ctypes.c_int
    I64P = ctypes.POINTER(ctypes.c_int64)
    L.crvpinn_default_opts.argtypes = [ctypes.POINTER(Opts)]
    L.crvpinn_create.argtypes = [ctypes.POINTER(P), I, I, ctypes.POINTER(I), F, F, F, F, ctypes.POINTER(Opts)]
    L.crvpinn_set_saturation.argtypes = [P, F]
    L.crvpinn_set_saturation_device.argtypes = [P, P]
    L.crvpinn_pretrain.argtypes = [P, I, D]
    L.crvpinn_step.argtypes = [P, I, D]
    L.crvpinn_eval.argtypes = [P, F]
    L.crvpinn_loss_grad.argtypes = [P, D, F]
    L.crvpinn_eval_points.argtypes = [P, ctypes.c_long, F, F]
    L.crvpinn_direct_solve.argtypes = [P, ctypes.c_double, I, F, ctypes.POINTER(ctypes.c_int), D]
    L.crvpinn_get_intermediates.argtypes = [P, F, F, F, F]
    L.crvpinn_num_params.restype = ctypes.c_size_t
    L.crvpinn_num_params.argtypes = [P]
    L.crvpinn_get_params.argtypes = [P, F]
    L.crvpinn_set_params.argtypes = [P, F]
    L.crvpinn_get_adam.argtypes = [P, F, F, I64P]
    L.crvpinn_set_adam.argtypes = [P, F, F, ctypes.c_int64]
    L.crvpinn_set_profiling.argtypes = [P, I]
    L.crvpinn_get_profile.argtypes = [P, D, I64P, I]
    L.crvpinn_launches_per_iter.argtypes = [P]
    L.crvpinn_stream.restype = P
    L.crvpinn_stream.argtypes = [P]
    L.crvpinn_last_error.restype = ctypes.c_char_p
    L.crvpinn_last_error.argtypes = [P]
    L.crvpinn_destroy.argtypes = [P]
    L.crvpinn_shard_tiles.argtypes = [I, I, I, ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long)]
    L.crvpinn_nccl_unique_id.argtypes = [ctypes.POINTER(ctypes.c_ubyte)]
    L.crvpinn_shard_forward.argtypes = [P, F]
    L.crvpinn_shard_backward.argtypes = [P, F, D, F]
    for name in ["crvpinn_create", "crvpinn_set_saturation", "crvpinn_set_saturation_device", "crvpinn_pretrain",
                 "crvpinn_step", "crvpinn_eval", "crvpinn_eval_points", "crvpinn_direct_solve", "crvpinn_loss_grad",
                 "crvpinn_get_intermediates",
                 "crvpinn_get_params", "crvpinn_set_params", "crvpinn_get_adam", "crvpinn_set_adam",
                 "crvpinn_set_profiling", "crvpinn_get_profile", "crvpinn_launches_per_iter",
                 "crvpinn_shard_tiles", "crvpinn_nccl_unique_id", "crvpinn_shard_forward", "crvpinn_shard_backward"]:
        getattr(L, name).restype = I
    L.crvpinn_iga_create.argtypes = [ctypes.POINTER(P), I, I, I]
    L.crvpinn_iga_create.restype = I
    L.crvpinn_iga_num_basis.argtypes = [P]
    L.crvpinn_iga_num_basis.restype = I
    L.crvpinn_iga_num_quad_points.argtypes = [P]
    L.crvpinn_iga_num_quad_points.restype = ctypes.c_long
    L.crvpinn_iga_quad_points.argtypes = [P, F]
    L.crvpinn_iga_project.argtypes = [P, F, F]
    L.crvpinn_iga_saturation_step.argtypes = [P, F, F, F, F, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_double, ctypes.c_double, F]
    L.crvpinn_iga_eval.argtypes = [P, F, ctypes.c_long, F, F, F]
    L.crvpinn_iga_last_ms.argtypes = [P]
    L.crvpinn_iga_last_ms.restype = ctypes.c_double
    L.crvpinn_iga_last_error.argtypes = [P]
    L.crvpinn_iga_last_error.restype = ctypes.c_char_p
    L.crvpinn_iga_destroy.argtypes = [P]
    for name in ["crvpinn_iga_quad_points", "crvpinn_iga_project", "crvpinn_iga_saturation_step", "crvpinn_iga_eval"]:
        getattr(L, name).restype = I
    _lib = L
    return L


def _f32(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if n is not None and a.size != n:
        raise ValueError(f"expected {n} values, got {a.size}")
    return a


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def default_opts() -> Opts:
    o = Opts()
    load().crvpinn_default_opts(ctypes.byref(o))
    return o


def shard_tiles(N: int, rank: int, world: int):
    """(tile0, ntiles): shard `rank` of `world` over the N*N/128 MLP tiles (crvpinn_shard_tiles; host only)."""
    t0, nt = ctypes.c_long(), ctypes.c_long()
    rc = load().crvpinn_shard_tiles(int(N), int(rank), int(world), ctypes.byref(t0), ctypes.byref(nt))
    if rc != 0:
        raise CrvpinnError(rc, load().crvpinn_last_error(None).decode())
    return int(t0.value), int(nt.value)


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for Crvpinn(shard=..., nccl_id=...)."""
    buf = (ctypes.c_ubyte * 128)()
    rc = load().crvpinn_nccl_unique_id(buf)
    if rc != 0:
        raise CrvpinnError(rc, load().crvpinn_last_error(None).decode())
    return bytes(buf)


def share_nccl_id(group=None, src: int = 0, make_id=None) -> bytes:
    """Rank `src` of the torch.distributed group creates the id, every rank returns it (plumbing only)."""
    import torch.distributed as dist
    obj = [(make_id or nccl_unique_id)() if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


class Crvpinn:
    """One CRVPINN problem on one GPU (wraps crvpinn_ctx). shard=(rank, world) runs this GPU's share of
    the MLP points; with nccl_id the context exchanges u and the gradient itself."""

    def __init__(self, N: int, widths: Sequence[int], K, S, f, theta0=None, *, precision: int = PREC_TENSOR,
                 lr: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 mobility_ratio: Optional[float] = None, seed: int = 0, stream: Optional[int] = None,
                 device: int = 0, gravity: float = 0.0, density_ratio: Optional[float] = None,
                 shard: Optional[Tuple[int, int]] = None, nccl_id: Optional[bytes] = None):
        L = load()
        self.N = int(N)
        self.widths = tuple(int(w) for w in widths)
        nn = (self.N + 1) ** 2
        o = default_opts()
        o.lr, o.beta1, o.beta2, o.eps = lr, beta1, beta2, eps
        if mobility_ratio is not None:
            o.mobility_ratio = mobility_ratio
        o.precision, o.seed, o.device = precision, seed, device
        o.gravity = gravity
        if density_ratio is not None:
            o.density_ratio = density_ratio
        o.stream = stream
        if shard is not None:
            o.shard_rank, o.shard_world = int(shard[0]), int(shard[1])
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes")
            o.nccl = 1
            ctypes.memmove(o.nccl_id, nccl_id, 128)
        self.shard = (o.shard_rank, o.shard_world)
        w = (ctypes.c_int * len(self.widths))(*self.widths)
        K, S, f = _f32(K, nn), _f32(S, nn), _f32(f, nn)
        wd = self.widths
        n_params = sum(wd[l + 1] * (wd[l] + 1) for l in range(len(wd) - 1))
        th = None if theta0 is None else _f32(theta0, n_params)   # the C side reads exactly n_params floats
        h = ctypes.c_void_p()
        rc = L.crvpinn_create(ctypes.byref(h), self.N, len(self.widths), w, _fp(K), _fp(S), _fp(f),
                              None if th is None else _fp(th), ctypes.byref(o))
        if rc != 0:
            raise CrvpinnError(rc, L.crvpinn_last_error(None).decode())
        self._h = h
        self.precision = precision
        self.np = int(L.crvpinn_num_params(h))

    def _check(self, rc):
        if rc != 0:
            raise CrvpinnError(rc, load().crvpinn_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            if load is None:          # interpreter shutdown: module globals already cleared
                return
            load().crvpinn_destroy(self._h)
            self._h = None

    __del__ = close

    # ---- the boundary calls (same names as include/crvpinn.h)
    def set_saturation(self, S):
        self._check(load().crvpinn_set_saturation(self._h, _fp(_f32(S, (self.N + 1) ** 2))))

    def set_saturation_device(self, ptr: int):
        self._check(load().crvpinn_set_saturation_device(self._h, ctypes.c_void_p(ptr)))

    def pretrain(self, n_iters: int, history: bool = True):
        hist = np.empty(n_iters) if history else None
        self._check(load().crvpinn_pretrain(self._h, int(n_iters),
                                            None if hist is None else hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return hist

    def step(self, n_adam: int = 100, history: bool = True):
        hist = np.empty(n_adam) if history else None
        self._check(load().crvpinn_step(self._h, int(n_adam),
                                        None if hist is None else hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return hist

    def eval(self) -> np.ndarray:
        out = np.empty((self.N + 1) ** 2, np.float32)
        self._check(load().crvpinn_eval(self._h, _fp(out)))
        return out

    def eval_points(self, xy) -> np.ndarray:
        """p(x, y) = cutoff * net at arbitrary points; xy: (n, 2) array-like -> (n,) float32."""
        xy = np.ascontiguousarray(np.asarray(xy, dtype=np.float32).reshape(-1, 2))
        out = np.empty(xy.shape[0], dtype=np.float32)
        if xy.shape[0]:
            self._check(load().crvpinn_eval_points(self._h, int(xy.shape[0]), _fp(xy), _fp(out)))
        return out

    def direct_solve(self, rtol: float = 1e-5, max_iter: int = 20000):
        """u with A(alpha) u = b (Gram-preconditioned CG) -> (u lattice (N+1)^2, iterations, rel. residual)."""
        u = np.empty((self.N + 1) ** 2, dtype=np.float32)
        it, rel = ctypes.c_int(0), ctypes.c_double(0.0)
        self._check(load().crvpinn_direct_solve(self._h, float(rtol), int(max_iter), _fp(u), ctypes.byref(it),
                                                ctypes.byref(rel)))
        return u, int(it.value), float(rel.value)

    def loss_grad(self, grad: bool = True):
        loss = ctypes.c_double()
        g = np.empty(self.np, np.float32) if grad else None
        self._check(load().crvpinn_loss_grad(self._h, ctypes.byref(loss), None if g is None else _fp(g)))
        return (loss.value, g) if grad else loss.value

    def shard_forward(self) -> np.ndarray:
        """This shard's points of u (zero elsewhere), lattice (N+1)^2; no collective."""
        out = np.empty((self.N + 1) ** 2, np.float32)
        self._check(load().crvpinn_shard_forward(self._h, _fp(out)))
        return out

    def shard_backward(self, u_full):
        """(loss of u_full, this shard's share of the gradient); no collective."""
        u = _f32(u_full, (self.N + 1) ** 2)
        loss = ctypes.c_double()
        g = np.empty(self.np, np.float32)
        self._check(load().crvpinn_shard_backward(self._h, _fp(u), ctypes.byref(loss), _fp(g)))
        return loss.value, g

    def intermediates(self):
        nn, n2 = (self.N + 1) ** 2, (self.N - 1) ** 2
        u, r, q, gu = (np.empty(nn, np.float32), np.empty(n2, np.float32), np.empty(n2, np.float32),
                       np.empty(nn, np.float32))
        self._check(load().crvpinn_get_intermediates(self._h, _fp(u), _fp(r), _fp(q), _fp(gu)))
        return dict(u=u, res=r, q=q, gu=gu)

    @property
    def theta(self) -> np.ndarray:
        out = np.empty(self.np, np.float32)
        self._check(load().crvpinn_get_params(self._h, _fp(out)))
        return out

    @theta.setter
    def theta(self, th):
        self._check(load().crvpinn_set_params(self._h, _fp(_f32(th, self.np))))

    def adam_state(self):
        m, v, t = np.empty(self.np, np.float32), np.empty(self.np, np.float32), ctypes.c_int64()
        self._check(load().crvpinn_get_adam(self._h, _fp(m), _fp(v), ctypes.byref(t)))
        return m, v, int(t.value)

    def set_adam_state(self, m, v, t: int):
        self._check(load().crvpinn_set_adam(self._h, _fp(_f32(m, self.np)), _fp(_f32(v, self.np)), int(t)))

    def set_profiling(self, on: bool):
        self._check(load().crvpinn_set_profiling(self._h, 1 if on else 0))

    def profile(self, reset: bool = False):
        ms = (ctypes.c_double * 4)()
        n = ctypes.c_int64()
        self._check(load().crvpinn_get_profile(self._h, ms, ctypes.byref(n), 1 if reset else 0))
        return list(ms), int(n.value)

    @property
    def launches_per_iter(self) -> int:
        return int(load().crvpinn_launches_per_iter(self._h))

    @property
    def stream(self) -> int:
        return int(load().crvpinn_stream(self._h) or 0)


class Iga:
    """Tensor-product B-spline space on [0,1]^2 on the GPU (crvpinn_iga): the IGA-ADS saturation step
    (SURVEY.md §8(f) f3). Coefficients are (nb, nb) float32 arrays indexed [l][k] (row = y)."""

    def __init__(self, n_elements: int, degree: int = 2, device: int = 0):
        L = load()
        h = ctypes.c_void_p()
        rc = L.crvpinn_iga_create(ctypes.byref(h), int(n_elements), int(degree), int(device))
        if rc != 0:
            raise CrvpinnError(rc, "crvpinn_iga_create failed")
        self._h = h
        self.ne, self.r = int(n_elements), int(degree)
        self.nb = int(L.crvpinn_iga_num_basis(h))
        self.nq = int(L.crvpinn_iga_num_quad_points(h))

    def close(self):
        if getattr(self, "_h", None):
            if load is None:
                return
            load().crvpinn_iga_destroy(self._h)
            self._h = None

    __del__ = close

    def _check(self, rc):
        if rc != 0:
            raise CrvpinnError(rc, load().crvpinn_iga_last_error(self._h).decode())

    def quad_points(self) -> np.ndarray:
        out = np.empty((self.nq, 2), dtype=np.float32)
        self._check(load().crvpinn_iga_quad_points(self._h, _fp(out)))
        return out

    def project(self, fq) -> np.ndarray:
        fq = _f32(fq, self.nq)
        out = np.empty((self.nb, self.nb), dtype=np.float32)
        self._check(load().crvpinn_iga_project(self._h, _fp(fq), _fp(out)))
        return out

    def saturation_step(self, S, P, K_elem, q_elem, tau: float, phi: float = 1.0, mobility_ratio: float = 25.35 / 3.95,
                        density_ratio: float = 479.0 / 1045.0, gravity: float = 0.0) -> np.ndarray:
        n2, e2 = self.nb * self.nb, self.ne * self.ne
        S, P, K, q = _f32(S, n2), _f32(P, n2), _f32(K_elem, e2), _f32(q_elem, e2)
        out = np.empty((self.nb, self.nb), dtype=np.float32)
        self._check(load().crvpinn_iga_saturation_step(self._h, _fp(S), _fp(P), _fp(K), _fp(q), float(tau), float(phi),
                                                       float(mobility_ratio), float(density_ratio), float(gravity),
                                                       _fp(out)))
        return out

    def eval(self, coef, xy, grad: bool = False):
        C = _f32(coef, self.nb * self.nb)
        xy = np.ascontiguousarray(np.asarray(xy, dtype=np.float32).reshape(-1, 2))
        val = np.empty(xy.shape[0], dtype=np.float32)
        g = np.empty((xy.shape[0], 2), dtype=np.float32) if grad else None
        if xy.shape[0]:
            self._check(load().crvpinn_iga_eval(self._h, _fp(C), int(xy.shape[0]), _fp(xy), _fp(val),
                                                None if g is None else _fp(g)))
        return (val, g) if grad else val

    @property
    def last_ms(self) -> float:
        return float(load().crvpinn_iga_last_ms(self._h))
