"""A model of a PRECISION CLASS (not of any implementation): the oracle's Adam iteration with the
backward pass's per-point operands rounded to 11 significant bits.

TEST INFRASTRUCTURE ONLY, like the rest of oracle/: imported by tests/ and scripts/ that write
fixtures; never by the product package, which shares no code with it.

Why it exists (reading R28). north_star admits "TF32" arithmetic for the MLP
contractions. TF32 and fp16 operands both carry an 11-bit significand. Late in C3's pretraining
(§6 step 2; 2000 iterations) the gradient dLOSS/dtheta = sum_p (per-point terms)
is a sum whose terms cancel to ~1e-3 of their magnitudes, so rounding the per-point operands of
the backward (activations t in dW and in 1 - t^2, deltas Delta, weights W) to 11 bits changes the
gradient by O(1) at such points. A trajectory computed in that class is therefore a different
(noise-driven) trajectory of the same chaotic iteration, and its long-horizon statistics are
compared with this model's ensemble, not with the exact oracle's.

What it computes, step by step (the paper's order, as oracle/crvpinn_oracle.c):
  A1  u = 16x(1-x)y(1-y) net_theta(x, y) at the interior nodes, tanh MLP, fp64;
  A2-A5  RES, q = G^-1 RES, LOSS = RES^T q and dLOSS/du from the oracle itself
         (Oracle.loss_u, Oracle.residual_adjoint: Eqs. 25-28);
  A6  reverse mode through the MLP (the chain rule) in fp64 with, when bits=11,
      t, Delta and W rounded (round-to-nearest-even) to 11 significant bits wherever the backward
      multiplies with them; sums in fp64;
  A8  Adam from the oracle (Oracle.adam_step, reading R7).
With bits=None nothing is rounded and the model is the oracle's iteration itself (pinned in
tests/test_oracle_pins.py: gradient equal to Oracle.loss_grad to 1e-12, trajectory equal to
Oracle.train).
"""
from __future__ import annotations

import numpy as np

from . import Oracle


def round_sig(a: np.ndarray, bits: int = 11) -> np.ndarray:
    """Round to `bits` significant bits, round-to-nearest-even, at any magnitude (no exponent limits:
    the operand scales of the class keep fp16 values in range). bits = 11: fp16 / TF32;
    bits = 24: fp32."""
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)                               # a = m 2^e, |m| in [0.5, 1)
    return np.ldexp(np.rint(np.ldexp(m, bits)), e - bits)


class PrecisionModel:
    def __init__(self, N, widths, K, S, f, theta0, *, lr=1e-3, bits=11):
        self.o = Oracle(N, widths, K, S, f, theta0, lr=lr)
        self.N, self.widths, self.bits = int(N), tuple(int(w) for w in widths), bits
        i, j = np.meshgrid(np.arange(1, N), np.arange(1, N), indexing="xy")
        self.node = (j * (N + 1) + i).ravel()          # lattice index of every interior node
        self.x, self.y = (i / N).ravel(), (j / N).ravel()
        self.cut = 16.0 * self.x * (1 - self.x) * self.y * (1 - self.y)

    def _layers(self, th):
        out, off = [], 0
        ws = self.widths
        for l in range(len(ws) - 1):
            W = th[off:off + ws[l + 1] * ws[l]].reshape(ws[l + 1], ws[l])
            off += ws[l + 1] * ws[l]
            b = th[off:off + ws[l + 1]]
            off += ws[l + 1]
            out.append((W, b))
        return out

    def _r(self, a):
        return a if self.bits is None else round_sig(a, self.bits)

    def loss_grad(self):
        th = self.o.theta
        lay = self._layers(th)
        X = np.stack([self.x, self.y], 1)
        ts, a = [], X
        for W, b in lay[:-1]:
            a = np.tanh(a @ W.T + b)
            ts.append(a)
        Wo, bo = lay[-1]
        net = (a @ Wo.T + bo)[:, 0]
        u = np.zeros((self.N + 1) ** 2)
        u[self.node] = self.cut * net
        loss, _, q = self.o.loss_u(u)
        gu = self.o.residual_adjoint(2.0 * q)
        gbar = self.cut * gu[self.node]                  # dLOSS/dnet per point
        tr = [self._r(t) for t in ts]
        grads = [None] * (2 * len(lay))
        L = len(lay) - 1
        grads[2 * L] = (gbar[:, None] * tr[-1]).sum(0)[None, :]
        grads[2 * L + 1] = np.array([gbar.sum()])
        D = self._r(gbar[:, None] * Wo * (1.0 - tr[-1] ** 2))
        for l in range(L - 1, 0, -1):                     # W_l maps t_{l-1} -> z_l
            grads[2 * l] = D.T @ tr[l - 1]
            grads[2 * l + 1] = D.sum(0)
            D = self._r((D @ self._r(lay[l][0])) * (1.0 - tr[l - 1] ** 2))
        grads[0] = D.T @ X
        grads[1] = D.sum(0)
        return loss, np.concatenate([g.ravel() for g in grads])

    def train(self, n_iters: int) -> np.ndarray:
        hist = np.empty(n_iters)
        for k in range(n_iters):
            hist[k], g = self.loss_grad()
            self.o.adam_step(g)
        return hist
