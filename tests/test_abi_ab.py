"""ABI-level A/B: ONE ctypes driver calls the same C entry points (include/crvpinn.h)
of two libraries -- the CUDA product (paper_2604_20731_b200/libcrvpinn.so) and the fp64 CPU oracle
behind the same ABI (oracle/liboracle_abi.so, oracle/crvpinn_abi.c) -- on the same seeded inputs.

CPU tests (`-m "not gpu"`) pin the oracle ABI to the oracle itself (oracle.Oracle) and check that it
exports the §8(b) core calls the product header declares; the `gpu` tests run the A/B proper.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "crvpinn.h")
CORE = ["crvpinn_default_opts", "crvpinn_create", "crvpinn_set_saturation", "crvpinn_pretrain", "crvpinn_step",
        "crvpinn_eval", "crvpinn_loss_grad", "crvpinn_get_intermediates", "crvpinn_num_params",
        "crvpinn_get_params", "crvpinn_set_params", "crvpinn_get_adam", "crvpinn_last_error", "crvpinn_destroy"]


class Opts(ctypes.Structure):
    """crvpinn_opts as include/crvpinn.h documents it."""
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("mobility_ratio", ctypes.c_double), ("precision", ctypes.c_int),
                ("seed", ctypes.c_uint64), ("stream", ctypes.c_void_p), ("device", ctypes.c_int),
                ("gravity", ctypes.c_double), ("density_ratio", ctypes.c_double),
                ("shard_rank", ctypes.c_int), ("shard_world", ctypes.c_int), ("nccl", ctypes.c_int),
                ("nccl_id", ctypes.c_ubyte * 128)]


class AbiDriver:
    """The §8(b) calls through a bare C ABI; `path` selects the implementation."""

    def __init__(self, path, N, widths, K, S, f, theta0, precision=0, lr=1e-3):
        L = ctypes.CDLL(path)
        P, F, D = ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)
        L.crvpinn_default_opts.argtypes = [ctypes.POINTER(Opts)]
        L.crvpinn_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                     F, F, F, F, ctypes.POINTER(Opts)]
        for name, args in [("crvpinn_set_saturation", [P, F]), ("crvpinn_pretrain", [P, ctypes.c_int, D]),
                           ("crvpinn_step", [P, ctypes.c_int, D]), ("crvpinn_eval", [P, F]),
                           ("crvpinn_loss_grad", [P, D, F]), ("crvpinn_get_intermediates", [P, F, F, F, F]),
                           ("crvpinn_get_params", [P, F]), ("crvpinn_set_params", [P, F]),
                           ("crvpinn_get_adam", [P, F, F, ctypes.POINTER(ctypes.c_int64)])]:
            getattr(L, name).argtypes = args
            getattr(L, name).restype = ctypes.c_int
        L.crvpinn_num_params.argtypes = [P]
        L.crvpinn_num_params.restype = ctypes.c_size_t
        L.crvpinn_last_error.argtypes = [P]
        L.crvpinn_last_error.restype = ctypes.c_char_p
        L.crvpinn_destroy.argtypes = [P]
        self.L, self.N = L, N
        o = Opts()
        L.crvpinn_default_opts(ctypes.byref(o))
        o.precision, o.lr = precision, lr
        w = (ctypes.c_int * len(widths))(*widths)
        self.ctx = P()
        self._ok(L.crvpinn_create(ctypes.byref(self.ctx), N, len(widths), w, self._f(K), self._f(S), self._f(f),
                                  self._f(theta0), ctypes.byref(o)), None)
        self.np = int(L.crvpinn_num_params(self.ctx))

    @staticmethod
    def _f(a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        AbiDriver._keep = getattr(AbiDriver, "_keep", []) + [a]
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))

    def _ok(self, rc, ctx="self"):
        if rc != 0:
            raise RuntimeError(f"rc {rc}: {self.L.crvpinn_last_error(self.ctx if ctx else None)}")

    def loss_grad(self):
        loss = ctypes.c_double()
        g = np.zeros(self.np, np.float32)
        self._ok(self.L.crvpinn_loss_grad(self.ctx, ctypes.byref(loss), g.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return loss.value, g

    def step(self, n, pretrain=False):
        h = np.zeros(n, np.float64)
        fn = self.L.crvpinn_pretrain if pretrain else self.L.crvpinn_step
        rc = fn(self.ctx, n, h.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return rc, h

    def eval(self):
        p = np.zeros((self.N + 1) ** 2, np.float32)
        self._ok(self.L.crvpinn_eval(self.ctx, p.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return p

    def intermediates(self):
        nn, n2 = (self.N + 1) ** 2, (self.N - 1) ** 2
        u, r, q, gu = (np.zeros(k, np.float32) for k in (nn, n2, n2, nn))
        F = ctypes.POINTER(ctypes.c_float)
        self._ok(self.L.crvpinn_get_intermediates(self.ctx, *(a.ctypes.data_as(F) for a in (u, r, q, gu))))
        return u, r, q, gu

    def params(self):
        t = np.zeros(self.np, np.float32)
        self._ok(self.L.crvpinn_get_params(self.ctx, t.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return t

    def set_params(self, t):
        self._ok(self.L.crvpinn_set_params(self.ctx, self._f(t)))

    def adam(self):
        m, v = np.zeros(self.np, np.float32), np.zeros(self.np, np.float32)
        t = ctypes.c_int64()
        F = ctypes.POINTER(ctypes.c_float)
        self._ok(self.L.crvpinn_get_adam(self.ctx, m.ctypes.data_as(F), v.ctypes.data_as(F), ctypes.byref(t)))
        return m, v, t.value

    def set_saturation(self, S):
        self._ok(self.L.crvpinn_set_saturation(self.ctx, self._f(S)))

    def close(self):
        if self.ctx:
            self.L.crvpinn_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()


@pytest.fixture(scope="module")
def orc_abi():
    oracle.build()
    return oracle.LIB_ABI


def _problem(N=16, widths=(2, 32, 32, 1), seed=61):
    K, S, f = W.random_fields(N, seed)
    return N, widths, K, S, f, W.random_theta(widths, seed)


def test_oracle_abi_exports_the_core_calls(orc_abi):
    """The oracle library exports every §8(b) core call, and the product header declares each."""
    out = subprocess.check_output(["nm", "-D", "--defined-only", orc_abi]).decode()
    exported = set(re.findall(r" T (crvpinn_\w+)", out))
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    declared = set(re.findall(r"\b(crvpinn_[a-z_]+)\s*\(", text))
    for name in CORE:
        assert name in exported, name
        assert name in declared, name


def test_oracle_abi_equals_oracle(orc_abi):
    """Pin of the shim: through the ABI, LOSS / gradient / intermediates / 5-step history / eval and the
    Adam state equal oracle.Oracle's (the same fp64 functions; the ABI rounds its outputs to float32)."""
    N, widths, K, S, f, th = _problem()
    a = AbiDriver(orc_abi, N, widths, K, S, f, th)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    loss, g = a.loss_grad()
    rl, rg, it = ref.loss_grad(intermediates=True)
    assert loss == rl
    np.testing.assert_array_equal(g, rg.astype(np.float32))
    u, r, q, gu = a.intermediates()
    for x, key in ((u, "u"), (r, "res"), (q, "q"), (gu, "gu")):
        np.testing.assert_array_equal(x, np.asarray(it[key]).astype(np.float32))
    rc, h = a.step(5)
    assert rc == 0
    np.testing.assert_array_equal(h, ref.train(5))
    np.testing.assert_array_equal(a.params(), ref.theta.astype(np.float32))
    m, v, t = a.adam()
    rm, rv, rt = ref.adam_state()
    assert t == rt == 5
    np.testing.assert_array_equal(m, rm.astype(np.float32))
    np.testing.assert_array_equal(a.eval(), ref.forward().astype(np.float32))
    S2 = np.clip(S * 0.5 + 0.25, 0, 1).astype(np.float32)
    a.set_saturation(S2)
    ref.set_saturation(S2)
    assert a.loss_grad()[0] == ref.loss_grad()[0]
    a.close()


def test_oracle_abi_contract_errors(orc_abi):
    """EINVAL (N not a power of two), EDOMAIN (K <= 0), and ENONFINITE in the middle of a call with
    theta and the Adam state restored to their call-entry values (the ABI's contract)."""
    N, widths, K, S, f, th = _problem()
    with pytest.raises(RuntimeError, match="rc -1"):
        AbiDriver(orc_abi, 12, widths, K, S, f, th)
    Kb = K.copy()
    Kb[3] = 0.0
    with pytest.raises(RuntimeError, match="rc -5"):
        AbiDriver(orc_abi, N, widths, Kb, S, f, th)
    a = AbiDriver(orc_abi, N, widths, K, S, f, th, lr=1e300)   # update 1 sends theta to ~1e300: LOSS overflows
    t_entry, (m_entry, v_entry, n_entry) = a.params(), a.adam()
    rc, h = a.step(3)
    assert rc == -4 and np.isfinite(h[0]) and not np.isfinite(h[1])
    np.testing.assert_array_equal(a.params(), t_entry)
    m, v, n = a.adam()
    assert n == n_entry == 0
    np.testing.assert_array_equal(m, m_entry)
    np.testing.assert_array_equal(v, v_entry)
    a.close()


# ------------------------------------------------------------------ the A/B proper (GPU)
TOL = {0: (5e-3, 1e-2), 1: (1e-4, 1e-3)}   # north_star: (loss rel, gradient rel-L2), TF32 / fp32 class


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [pytest.param(1, id="fp32"), pytest.param(0, id="tensor")])
@pytest.mark.parametrize("case", ["C1", "N64"])
def test_abi_ab_product_vs_oracle(orc_abi, prec, case):
    """The same driver on both libraries: LOSS and gradient at theta0, the 20-step loss history, the
    state after it, a saturation update and eval -- the product within the north_star tolerances."""
    import paper_2604_20731_b200 as crv
    crv.load()
    if case == "C1":
        F = W.make_fields("C1")
        N, widths, K, S, f, th = F.workload.N, F.workload.widths, F.K, F.S, F.f, F.theta0
    else:
        N, widths, K, S, f, th = _problem(64, (2, 64, 64, 64, 1), 62)
    runs = [AbiDriver(p, N, widths, K, S, f, th, precision=prec) for p in (crv.LIB_PATH, orc_abi)]
    (lp, gp), (lo, go) = (r.loss_grad() for r in runs)
    tl, tg = TOL[prec]
    assert abs(lp - lo) <= tl * abs(lo)
    assert np.linalg.norm(gp - go) <= tg * np.linalg.norm(go)
    (rcp, hp), (rco, ho) = (r.step(20) for r in runs)
    assert rcp == rco == 0
    assert np.all(np.abs(hp - ho) <= 0.02 * np.abs(ho))
    assert runs[0].adam()[2] == runs[1].adam()[2] == 20
    S2 = np.clip(np.asarray(S) * 0.5 + 0.3, 0, 1).astype(np.float32)
    for r in runs:
        r.set_saturation(S2)
    (lp, _), (lo, _) = (r.loss_grad() for r in runs)
    assert abs(lp - lo) <= max(tl, 0.02) * abs(lo)
    pp, po = (r.eval() for r in runs)
    assert np.max(np.abs(pp - po)) <= (1e-4 if prec == 1 else 2e-3) * np.abs(po).max()
    for r in runs:
        r.close()
