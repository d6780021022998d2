"""Seeded synthetic inputs for the five CRVPINN workloads (C1..C5).

This module is shared by the oracle tests and the CUDA path. It holds NO arithmetic of
the method (no alpha, no residual, no Gram, no network evaluation): it only draws the
input fields K, S, f on the (N+1)x(N+1) node lattice and the initial network weights
theta0. Everything here is an input the paper takes as given (§6 step 1:
"Given the permeability map K, ..., the source terms q_w, q_g, ... the initial saturation").

The paper's own rasters (K1-K3) are figure files that are absent, so the
fields are synthetic stand-ins with the paper's shapes (unit-square lattice, heterogeneous K,
plume/front-shaped S, injection/production wells). Recipes are the readings Q12-Q15 of
SURVEY.md §8(c), restated in DESIGN.md §3.

Layout convention (SURVEY.md §8 notation): every field is float32, row-major
(N+1)x(N+1), F[j*(N+1)+i] at (x_i, y_j) = (i/N, j/N).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

# Table 1 of the paper. Only the viscosity ratio enters the build
# (reading Q10: alpha = K((1-S) + M S), M = mu_w/mu_g).
MU_G = 3.95e-5     # Pa s
MU_W = 25.35e-5    # Pa s
MOBILITY_RATIO = MU_W / MU_G   # 6.417721518987342


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    N: int                    # intervals per axis, h = 1/N (reading Q9)
    widths: tuple             # (2, w, ..., w, 1)
    lr: float
    n_adam: int               # Adam iterations per time step ("100 epochs")
    n_steps: int              # time steps (saturation updates)
    pretrain: int             # pretraining iterations before the steps
    description: str

    @property
    def n(self) -> int:
        return self.N - 1

    @property
    def points(self) -> int:
        return (self.N - 1) ** 2

    @property
    def n_params(self) -> int:
        w = self.widths
        return sum(w[i + 1] * w[i] + w[i + 1] for i in range(len(w) - 1))


WORKLOADS = {
    "C1": Workload("C1", 32, (2, 32, 32, 1), 1e-3, 100, 1, 0,
                   "32x32, K=1, S=0, q=2pi^2 sin sin (closed form p=sin sin)"),
    "C2": Workload("C2", 64, (2, 64, 64, 64, 1), 1e-3, 100, 1, 0,
                   "64x64, log-normal K (l=0.1, sigma=1), Gaussian plume S, +-1 point wells"),
    "C3": Workload("C3", 128, (2,) + (128,) * 4 + (1,), 1e-3, 100, 10, 2000,
                   "128x128, channelized K (1/0.1), smoothed random S, 2 wells; pretrain 2000"),
    "C4": Workload("C4", 256, (2,) + (128,) * 5 + (1,), 1e-3, 100, 10, 0,
                   "256x256, log-normal K (l=0.05, sigma=1.5), radial front S(t), t=1..10"),
    "C5": Workload("C5", 512, (2,) + (256,) * 5 + (1,), 1e-3, 100, 10, 0,
                   "512x512, log-normal K (l=0.03, sigma=2), front at t=10, 4+4 wells"),
}


def grid_xy(N: int):
    """Node coordinates (x_i, y_j) = (i/N, j/N) as (N+1)x(N+1) arrays indexed [j, i]."""
    c = np.arange(N + 1, dtype=np.float64) / N
    X, Y = np.meshgrid(c, c, indexing="xy")
    return X, Y


def _gaussian_field(rng: np.random.Generator, N: int, ell: float) -> np.ndarray:
    """Unit-variance Gaussian random field with covariance exp(-r^2/(2 ell^2)) (reading Q13).

    Separable Gaussian blur of N(0,1) white noise, kernel std s = ell/(sqrt(2) h) cells,
    truncated at +-4s, reflect padding, kernel normalised to unit l2 norm per axis.
    """
    h = 1.0 / N
    s = ell / (math.sqrt(2.0) * h)
    r = max(1, int(math.ceil(4.0 * s)))
    t = np.arange(-r, r + 1, dtype=np.float64)
    ker = np.exp(-t * t / (2.0 * s * s))
    ker /= math.sqrt(np.sum(ker * ker))
    noise = rng.standard_normal((N + 1, N + 1))
    pad = np.pad(noise, r, mode="reflect")
    # blur along x (axis 1) then y (axis 0)
    tmp = np.zeros((pad.shape[0], N + 1))
    for k, kv in enumerate(ker):
        tmp += kv * pad[:, k:k + N + 1]
    out = np.zeros((N + 1, N + 1))
    for k, kv in enumerate(ker):
        out += kv * tmp[k:k + N + 1, :]
    return out


def _wells(rng: np.random.Generator, N: int, count: int):
    """`count` distinct nodes drawn without replacement from [N/8, 7N/8]^2 (reading Q15)."""
    lo, hi = N // 8, (7 * N) // 8
    side = hi - lo + 1
    flat = rng.choice(side * side, size=count, replace=False)
    return [(lo + int(v % side), lo + int(v // side)) for v in flat]   # (i, j)


def _source_from_wells(N: int, injectors, producers) -> np.ndarray:
    """Unit-rate point wells: f = +-1/h^2 at the well node (reading Q12)."""
    f = np.zeros((N + 1, N + 1))
    h2inv = float(N * N)
    for (i, j) in injectors:
        f[j, i] += h2inv
    for (i, j) in producers:
        f[j, i] -= h2inv
    return f


def _front(N: int, centre, t: float) -> np.ndarray:
    """Radial front S = clip(1 - r/(0.05+0.02 t), 0, 1) (BASELINE.json configs[3])."""
    X, Y = grid_xy(N)
    cx, cy = centre[0] / N, centre[1] / N
    r = np.sqrt((X - cx) ** 2 + (Y - cy) ** 2)
    return np.clip(1.0 - r / (0.05 + 0.02 * t), 0.0, 1.0)


@dataclasses.dataclass
class Fields:
    """Inputs of one workload. S_steps[k] is the saturation for time step k."""
    workload: Workload
    K: np.ndarray              # float32 (N+1)^2
    f: np.ndarray              # float32 (N+1)^2
    S_steps: List[np.ndarray]  # float32 (N+1)^2 each
    theta0: np.ndarray         # float32 n_params

    @property
    def S(self) -> np.ndarray:
        return self.S_steps[0]


def make_fields(name: str, seed: Optional[int] = None, theta_seed: int = 0) -> Fields:
    """Generate the seeded inputs of workload `name` (field seed = config index, theta seed 0)."""
    w = WORKLOADS[name]
    N = w.N
    idx = int(name[1:])
    rng = np.random.Generator(np.random.PCG64(idx if seed is None else seed))
    X, Y = grid_xy(N)
    if name == "C1":
        K = np.ones((N + 1, N + 1))
        S_steps = [np.zeros((N + 1, N + 1))]
        f = 2.0 * math.pi ** 2 * np.sin(math.pi * X) * np.sin(math.pi * Y)
    elif name == "C2":
        K = np.exp(1.0 * _gaussian_field(rng, N, 0.1))
        c = rng.uniform(0.2, 0.8, size=2)
        S_steps = [0.8 * np.exp(-((X - c[0]) ** 2 + (Y - c[1]) ** 2) / (2 * 0.1 ** 2))]
        wl = _wells(rng, N, 2)
        f = _source_from_wells(N, wl[:1], wl[1:])
    elif name == "C3":
        K = np.full((N + 1, N + 1), 0.1)
        for _ in range(4):
            y0 = rng.uniform(0.1, 0.9)
            A = rng.uniform(0.05, 0.15)
            k = int(rng.integers(1, 4))
            phi = rng.uniform(0.0, 2 * math.pi)
            yc = y0 + A * np.sin(2 * math.pi * k * X + phi)
            K[np.abs(Y - yc) <= 4.0 / N] = 1.0
        S = rng.uniform(0.0, 1.0, size=(N + 1, N + 1))
        for _ in range(3):
            p = np.pad(S, 1, mode="edge")
            S = (p[1:-1, 1:-1] + p[:-2, 1:-1] + p[2:, 1:-1] + p[1:-1, :-2] + p[1:-1, 2:]) / 5.0
        S_steps = [S]
        wl = _wells(rng, N, 2)
        f = _source_from_wells(N, wl[:1], wl[1:])
    elif name == "C4":
        K = np.exp(1.5 * _gaussian_field(rng, N, 0.05))
        wl = _wells(rng, N, 2)
        f = _source_from_wells(N, wl[:1], wl[1:])
        S_steps = [_front(N, wl[0], t) for t in range(1, 11)]
    elif name == "C5":
        K = np.exp(2.0 * _gaussian_field(rng, N, 0.03))
        wl = _wells(rng, N, 8)
        f = _source_from_wells(N, wl[:4], wl[4:])
        S_steps = [_front(N, wl[0], 10.0)]
    else:
        raise KeyError(name)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32).reshape(-1)
    return Fields(w, f32(K), f32(f), [f32(s) for s in S_steps],
                  xavier_theta(w.widths, theta_seed))


def xavier_theta(widths, seed: int = 0) -> np.ndarray:
    """Xavier-uniform weights U(+-sqrt(6/(fan_in+fan_out))), biases 0 (reading Q6).

    Flattening order: W1 (row-major out x in), b1, ..., W_{L+1}, b_{L+1}.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    parts = []
    for i in range(len(widths) - 1):
        fin, fout = widths[i], widths[i + 1]
        a = math.sqrt(6.0 / (fin + fout))
        parts.append(rng.uniform(-a, a, size=(fout, fin)).reshape(-1))
        parts.append(np.zeros(fout))
    return np.concatenate(parts).astype(np.float32)


def random_theta(widths, seed: int, scale: float = 1.0) -> np.ndarray:
    """Xavier weights AND non-zero biases (used by tests so every parameter gets exercised)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    parts = []
    for i in range(len(widths) - 1):
        fin, fout = widths[i], widths[i + 1]
        a = math.sqrt(6.0 / (fin + fout)) * scale
        parts.append(rng.uniform(-a, a, size=(fout, fin)).reshape(-1))
        parts.append(rng.uniform(-0.1, 0.1, size=fout) * scale)
    return np.concatenate(parts).astype(np.float32)


def random_fields(N: int, seed: int, kmin: float = 0.2, kmax: float = 5.0):
    """Small random K in [kmin,kmax], S in [0,1], f ~ N(0,1) (parity-test inputs, tiny grids)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    K = rng.uniform(kmin, kmax, size=(N + 1) ** 2).astype(np.float32)
    S = rng.uniform(0.0, 1.0, size=(N + 1) ** 2).astype(np.float32)
    f = rng.standard_normal((N + 1) ** 2).astype(np.float32)
    return K, S, f


def theta_slices(widths):
    """(offset, shape) of every tensor in the flat theta: [(W1), (b1), ...]."""
    out, off = [], 0
    for i in range(len(widths) - 1):
        fin, fout = widths[i], widths[i + 1]
        out.append((off, (fout, fin)))
        off += fout * fin
        out.append((off, (fout,)))
        off += fout
    return out
