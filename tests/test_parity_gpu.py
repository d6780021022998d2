"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs. Tolerances are north_star's (BASELINE.json):
    loss relative error           <= 1e-4 (fp32 mode)  / 5e-3 (tensor mode, TF32 class)
    per-tensor gradient rel. L2   <= 1e-3 (fp32 mode)  / 1e-2 (tensor mode)
    final loss after 100 steps    within 2 %
Per-tensor rel-L2 uses a floor of 1e-3 x the global gradient norm for tensors whose own
gradient is (near) zero. Expensive oracle values (C3-C5) come from
tests/golden/*.npz written by scripts/make_golden.py, which calls only oracle/.
"""
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = {  # precision -> (loss rel, grad rel-L2)
    0: (5e-3, 1e-2),
    1: (1e-4, 1e-3),
}
PRECS = [pytest.param(1, id="fp32"), pytest.param(0, id="tensor")]
# element-wise u (A1) relative to max|u|. fp32 path: against the oracle's u. Tensor path: against the
# oracle's u at the network the tensor cores multiply with -- hidden GEMM weights rounded to 11
# significant bits (the fp16 copies; TF32 has the same significand) -- which the hi/lo-split forward
# evaluates to fp32 accuracy; the distance to the oracle at theta itself is then bounded by the
# oracle's own |u(theta~) - u(theta)|.
UTOL = {0: 2e-5, 1: 1e-5}


def class_theta(widths, th):
    """theta with the hidden-to-hidden weights rounded to 11 significant bits (round to nearest)."""
    from oracle.precision_model import round_sig
    out = np.array(th, dtype=np.float64)
    sl = W.theta_slices(widths)
    for l in range(1, len(widths) - 2):
        off, shape = sl[2 * l]
        n = int(np.prod(shape))
        out[off:off + n] = round_sig(out[off:off + n])
    return out


def check_u(prec, ref, widths, th, u, u_exact):
    """u of the GPU against the oracle (see UTOL); u_exact = the oracle's u at theta."""
    umax = np.abs(u_exact).max()
    if prec == 1:
        assert np.max(np.abs(u - u_exact)) <= UTOL[1] * umax
        return
    u_cls = ref.forward(theta=class_theta(widths, th))
    assert np.max(np.abs(u - u_cls)) <= UTOL[0] * umax, np.max(np.abs(u - u_cls)) / umax
    assert np.max(np.abs(u - u_exact)) <= np.max(np.abs(u_cls - u_exact)) + UTOL[0] * umax


@pytest.fixture(scope="module")
def crv():
    import paper_2604_20731_b200 as m
    from paper_2604_20731_b200 import build
    build.build()
    m.load()
    return m


def grad_errors(widths, g, ref):
    gnorm = np.linalg.norm(ref)
    out = []
    for off, shape in W.theta_slices(widths):
        n = int(np.prod(shape))
        a, b = g[off:off + n].astype(np.float64), ref[off:off + n].astype(np.float64)
        out.append(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-3 * gnorm))
    return np.array(out)


def _golden(name, kind):
    path = os.path.join(GOLDEN, f"{name}_{kind}.npz")
    if not os.path.exists(path):
        pytest.skip(f"missing fixture {path} (scripts/make_golden.py)")
    return np.load(path)


# ------------------------------------------------------------------ per-step intermediates
@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("N,widths,seed", [(16, (2, 32, 1), 0), (32, (2, 32, 32, 1), 1),
                                           (64, (2, 64, 64, 64, 1), 2), (32, (2, 128, 128, 1), 3),
                                           (16, (2, 256, 256, 1), 4), (64, (2, 256, 256, 256, 1), 5),
                                           (128, (2, 96, 96, 1), 6)])
def test_intermediates_vs_oracle(crv, prec, N, widths, seed):
    """u (A1), RES (A2), q (A3), LOSS (A4), dLOSS/du (A5), grads (A6/A7) at a random theta."""
    if prec == 0 and len(widths) < 4:
        pytest.skip("tensor path needs >= 2 hidden layers (one hidden GEMM)")
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    rl, rg, it = ref.loss_grad(intermediates=True)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec)
    loss, grad = g.loss_grad()
    im = g.intermediates()
    tl, tg = TOL[prec]
    check_u(prec, ref, widths, th, im["u"], it["u"])
    U = im["u"].reshape(N + 1, N + 1)
    assert np.all(U[0] == 0) and np.all(U[-1] == 0) and np.all(U[:, 0] == 0) and np.all(U[:, -1] == 0)
    # RES/q from the GPU's own u isolate the stencil and Gram kernels from the network
    r_own, q_own = ref.residual(im["u"]), ref.gram_solve(im["res"])
    assert np.max(np.abs(im["res"] - r_own)) <= 1e-5 * np.abs(r_own).max()
    assert np.max(np.abs(im["q"] - q_own)) <= 1e-5 * np.abs(q_own).max()
    gu_own = ref.residual_adjoint(2.0 * im["q"].astype(np.float64))
    mask = np.zeros((N + 1, N + 1))
    mask[1:-1, 1:-1] = 1
    gu_own *= mask.reshape(-1)
    assert np.max(np.abs(im["gu"] - gu_own)) <= 1e-5 * np.abs(gu_own).max()
    assert abs(loss - rl) <= tl * abs(rl)
    assert grad_errors(widths, grad, rg).max() <= tg


# ------------------------------------------------------------------ the five workloads at theta0
def _ref_theta0(name):
    F = W.make_fields(name)
    w = F.workload
    if name in ("C1", "C2"):
        o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
        loss, g, it = o.loss_grad(intermediates=True)
        return F, loss, g, it["u"]
    z = _golden(name, "theta0")
    return F, float(z["loss0"]), z["grad0"], z["u0"]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_workload_theta0_parity(crv, prec, name):
    F, rl, rg, ru = _ref_theta0(name)
    w = F.workload
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=prec, lr=w.lr)
    loss, grad = g.loss_grad()
    tl, tg = TOL[prec]
    assert abs(loss - rl) <= tl * abs(rl), (loss, rl)
    errs = grad_errors(w.widths, grad, rg)
    assert errs.max() <= tg, errs
    u = g.intermediates()["u"]
    o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr, factor_gram=False)
    check_u(prec, o, w.widths, F.theta0, u, ru)


# ------------------------------------------------------------------ 100 Adam steps
def _ref_traj(name):
    F = W.make_fields(name)
    w = F.workload
    if name in ("C1", "C2"):
        o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
        hist = o.train(100)
        return F, hist, o.loss_grad()[0]
    z = _golden(name, "traj100")
    return F, z["hist"], float(z["final_loss"])


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_workload_100_steps(crv, prec, name):
    F, rhist, rfinal = _ref_traj(name)
    w = F.workload
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=prec, lr=w.lr)
    hist = g.step(100)
    final = g.loss_grad(grad=False)
    assert abs(final - rfinal) <= 0.02 * abs(rfinal), (final, rfinal)
    assert abs(hist[0] - rhist[0]) <= TOL[prec][0] * abs(rhist[0])
    assert np.all(np.abs(hist - rhist) <= 0.02 * np.abs(rhist) + 1e-3 * np.abs(rhist).max())


def _ulp_perturbed(theta0, seed):
    """theta0 with every entry moved one fp32 ulp up or down (seeded signs); the recipe of
    scripts/c3_sensitivity.py, which wrote the oracle's perturbed fixtures."""
    t0 = np.asarray(theta0, dtype=np.float32)
    rng = np.random.default_rng(seed)
    return np.nextafter(t0, np.where(rng.random(t0.shape) < 0.5, -np.inf, np.inf).astype(np.float32))


def _ensemble(pattern, n=5):
    paths = [os.path.join(GOLDEN, pattern.format(s)) for s in range(n)]
    missing = [p for p in paths if not os.path.exists(p)]
    if missing:
        pytest.skip(f"missing fixtures {missing} (scripts/oracle_runs.py)")
    return [np.load(p)["hist"] for p in paths]


@pytest.mark.parametrize("prec", PRECS)
def test_c3_schedule_pretrain_and_updates(crv, prec):
    """C3's schedule (BASELINE.json configs[2]; §6 steps 2 and 7): pretraining of
    2000 Adam iterations, then 10 updates of 100 (fixed S), warm-started -- 3000 iterations in all.
    After a few hundred iterations the iteration is chaotic (R22: the oracle from theta0
    moved by one fp32 ulp leaves its own unperturbed run by > 2 % at iteration 388), so:
    (a) pointwise over the first 200 iterations against the oracle (the 100-step tolerance);
    (b) ensembles of 5 runs (theta0 + 4 ulp-perturbed starts) on both sides against the oracle's
        (tests/golden/C3_run3000_s*.npz): in each window the two ensemble means must agree within the
        sum of the two ensembles' spreads (a spread = the largest deviation of a member's window mean
        from its ensemble's mean), i.e. 2x their average spread (reading R22). The tensor path's window
        means are compared with the envelope of the oracle's ensemble and the 11-bit precision-class
        model's (tests/golden/C3_model11_run3000_s*.npz), each widened by its own spread, plus the
        tensor path's spread (reading R28: the 11-bit backward shifts these statistics by up to the
        model's -3.6 ... -29 %)."""
    F = W.make_fields("C3")
    w = F.workload
    runs = []
    for seed in range(5):
        th = F.theta0 if seed == 0 else _ulp_perturbed(F.theta0, seed)
        g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, th, precision=prec, lr=w.lr)
        runs.append(np.concatenate([g.pretrain(w.pretrain)] + [g.step(w.n_adam) for _ in range(w.n_steps)]))
        g.close()
    assert len(runs[0]) == 3000
    rhist = _golden("C3", "traj2000")["hist"]
    hist = runs[0]
    assert abs(hist[0] - rhist[0]) <= TOL[prec][0] * abs(rhist[0])
    dev = np.abs(hist[:200] - rhist[:200]) / (np.abs(rhist[:200]) + 1e-3 * np.abs(rhist).max())
    assert dev.max() <= 0.02, (int(dev.argmax()), float(dev.max()))
    ref = _ensemble("C3_run3000_s{}.npz")
    # the tensor path is an 11-bit (fp16 / TF32 class) backward (R28): its reference is the envelope of
    # the exact oracle's ensemble and the 11-bit class model's (oracle/precision_model.py, pinned by P21)
    refs = [ref] if prec == 1 else [ref, _ensemble("C3_model11_run3000_s{}.npz")]
    for a, b in ((900, 1100), (1800, 2000), (2400, 2600), (2800, 3000)):
        ours = np.array([r[a:b].mean() for r in runs])
        sp = np.max(np.abs(ours - ours.mean()))
        lo = min(np.mean([r[a:b].mean() for r in e]) - np.max(np.abs([r[a:b].mean() for r in e] -
                 np.mean([r[a:b].mean() for r in e]))) for e in refs) - sp
        hi = max(np.mean([r[a:b].mean() for r in e]) + np.max(np.abs([r[a:b].mean() for r in e] -
                 np.mean([r[a:b].mean() for r in e]))) for e in refs) + sp
        assert lo <= ours.mean() <= hi, ((a, b), ours.mean(), lo, hi)


@pytest.mark.parametrize("prec", PRECS)
def test_c4_schedule_10x100(crv, prec):
    """C4's full schedule (BASELINE.json configs[3]; §6 step 7 on the current S^n):
    10 time steps of 100 Adam iterations with warm-started weights and Adam state, the saturation
    front S(t) advanced between steps (crvpinn_set_saturation, step A0), against the oracle's run of
    the same schedule (tests/golden/C4_sched10x100.npz, scripts/oracle_runs.py c4sched): every
    step's loss history within the 100-step tolerance, and the loss at the end of every step."""
    z = _golden("C4", "sched10x100")
    F = W.make_fields("C4")
    w = F.workload
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S_steps[0], F.f, F.theta0, precision=prec, lr=w.lr)
    for k in range(w.n_steps):
        if k > 0:
            g.set_saturation(F.S_steps[k])
        hist = g.step(w.n_adam)
        rh = z["hist"][k]
        assert abs(hist[0] - rh[0]) <= 0.02 * abs(rh[0]), (k, hist[0], rh[0])
        assert np.all(np.abs(hist - rh) <= 0.02 * np.abs(rh) + 1e-3 * np.abs(rh).max()), k
        end = g.loss_grad(grad=False)
        assert abs(end - z["step_end"][k]) <= 0.02 * abs(z["step_end"][k]), (k, end, z["step_end"][k])


@pytest.mark.parametrize("prec", PRECS)
def test_c5_schedule(crv, prec):
    """C5's schedule (BASELINE.json configs[4]: 10 time steps of 100 Adam iterations on the fixed
    S of the t = 10 front; §6 step 7 with warm-started weights and Adam state),
    the time steps the oracle fixture holds (tests/golden/C5_sched.npz, scripts/oracle_runs.py
    c5sched: ~1 h of 8-core fp64 per step, `steps_done` of the 10): the same per-step bounds as
    C4's schedule test."""
    z = _golden("C5", "sched")
    F = W.make_fields("C5")
    w = F.workload
    n = int(z["steps_done"])
    if n < 2:
        pytest.skip(f"the fixture holds {n} time step(s); the warm-started schedule needs >= 2")
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=prec, lr=w.lr)
    for k in range(n):
        hist = g.step(w.n_adam)
        rh = z["hist"][k]
        assert abs(hist[0] - rh[0]) <= 0.02 * abs(rh[0]), (k, hist[0], rh[0])
        assert np.all(np.abs(hist - rh) <= 0.02 * np.abs(rh) + 1e-3 * np.abs(rh).max()), k
        end = g.loss_grad(grad=False)
        assert abs(end - z["step_end"][k]) <= 0.02 * abs(z["step_end"][k]), (k, end, z["step_end"][k])


# ------------------------------------------------------------------ semantics and edge cases
def test_step_composition_and_determinism(crv):
    """step(30)+step(70) == step(100) bitwise (Adam state persists, R8); runs are deterministic."""
    F = W.make_fields("C2")
    w = F.workload
    runs = []
    for split in [(100,), (30, 70), (100,)]:
        g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=1)
        hs = [g.step(k) for k in split]
        runs.append((np.concatenate(hs), g.theta, g.adam_state()))
    for h, th, (m, v, t) in runs[1:]:
        np.testing.assert_array_equal(h, runs[0][0])
        np.testing.assert_array_equal(th, runs[0][1])
        assert t == 100


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_step_run_to_run_bitwise(crv, name):
    """The graph step path is deterministic at full size: fresh contexts running step(20) give
    bit-identical loss histories and parameters (C4: backward chain with side-stream reductions; C5:
    per-GEMM backward, reductions after the last GEMM -- with side-stream reductions beside the GEMMs
    about one run in five differed)."""
    F = W.make_fields(name)
    w = F.workload
    runs = []
    for _ in range(4):
        g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
        runs.append((g.step(20), g.theta.copy()))
        g.close()
    for h, th in runs[1:]:
        np.testing.assert_array_equal(h, runs[0][0])
        np.testing.assert_array_equal(th, runs[0][1])


@pytest.mark.parametrize("prec", PRECS)
def test_set_saturation_matches_oracle(crv, prec):
    F = W.make_fields("C4")
    N = 32
    K, S, f = W.random_fields(N, 21)
    widths = (2, 64, 64, 1)
    th = W.random_theta(widths, 21)
    S2 = np.clip(S * 0.5 + 0.3, 0, 1).astype(np.float32)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    ref.set_saturation(S2)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec)
    g.set_saturation(S2)
    rl, rg = ref.loss_grad()
    loss, grad = g.loss_grad()
    assert abs(loss - rl) <= TOL[prec][0] * rl
    assert grad_errors(widths, grad, rg).max() <= TOL[prec][1]


def test_set_saturation_device_matches_host(crv):
    """crvpinn_set_saturation_device (the bench's device-resident S update) and the host call give the
    same alpha and RHS: 5 Adam steps after each update agree bit for bit, with and without gravity."""
    import torch
    N, widths, seed = 64, (2, 64, 64, 64, 1), 36
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    S2 = W.random_fields(N, seed + 1)[1]
    for Gr in (0.0, 0.7):
        a = crv.Crvpinn(N, widths, K, S, f, th, gravity=Gr)
        b = crv.Crvpinn(N, widths, K, S, f, th, gravity=Gr)
        a.set_saturation(S2)
        dS = torch.from_numpy(np.ascontiguousarray(S2, dtype=np.float32)).cuda()
        torch.cuda.synchronize()
        b.set_saturation_device(dS.data_ptr())
        np.testing.assert_array_equal(a.step(5), b.step(5))
        np.testing.assert_array_equal(a.theta, b.theta)


def test_eval_boundary_and_values(crv):
    N, widths = 32, (2, 64, 64, 1)
    K, S, f = W.random_fields(N, 5)
    th = W.random_theta(widths, 5)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=1)
    p = g.eval().reshape(N + 1, N + 1)
    assert np.all(p[0] == 0) and np.all(p[-1] == 0) and np.all(p[:, 0] == 0) and np.all(p[:, -1] == 0)
    ref = oracle.Oracle(N, widths, K, S, f, th, factor_gram=False).forward().reshape(N + 1, N + 1)
    assert np.max(np.abs(p - ref)) <= 1e-5 * np.abs(ref).max()


def test_nonfinite_restores_state(crv):
    N, widths = 16, (2, 32, 1)
    K, S, f = W.random_fields(N, 6)
    th = W.random_theta(widths, 6)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=1)
    g.step(5)
    th5, (m5, v5, t5) = g.theta, g.adam_state()
    bad = th5.copy()
    bad[0] = np.nan
    g.theta = bad
    with pytest.raises(crv.CrvpinnError) as ei:
        g.step(10)
    assert ei.value.code == crv.CRVPINN_ENONFINITE
    after = g.theta
    assert np.isnan(after[0]) and np.array_equal(after[1:], bad[1:])
    m, v, t = g.adam_state()
    assert t == t5 and np.array_equal(m, m5) and np.array_equal(v, v5)


@pytest.mark.parametrize("prec", PRECS)
def test_nonfinite_mid_call_restores_computation(crv, prec):
    """A divergence after several Adam steps of one call (lr = 1e38: the first update moves every
    weight by ~1e38, the next forward overflows): ENONFINITE, and the context computes exactly as at
    call entry afterwards -- theta, the Adam state and, on the tensor path, the fp16 weight copies
    the kernels read (rewritten by every Adam step of the call) are all restored."""
    N, widths = 32, (2, 64, 64, 64, 1)
    K, S, f = W.random_fields(N, 8)
    th = W.random_theta(widths, 8)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec, lr=1e38)
    l0, g0 = g.loss_grad()
    p0 = g.eval()
    with pytest.raises(crv.CrvpinnError) as ei:
        g.step(10)
    assert ei.value.code == crv.CRVPINN_ENONFINITE
    assert np.array_equal(g.theta, th)
    m, v, t = g.adam_state()
    assert t == 0 and not np.any(m) and not np.any(v)
    l1, g1 = g.loss_grad()
    assert l1 == l0 and np.array_equal(g1, g0)
    assert np.array_equal(g.eval(), p0)


def test_checkpoint_roundtrip(crv):
    N, widths = 32, (2, 32, 32, 1)
    K, S, f = W.random_fields(N, 7)
    th = W.random_theta(widths, 7)
    a = crv.Crvpinn(N, widths, K, S, f, th, precision=1)
    a.step(20)
    b = crv.Crvpinn(N, widths, K, S, f, None, precision=1)
    b.theta = a.theta
    b.set_adam_state(*a.adam_state())
    np.testing.assert_array_equal(a.step(15), b.step(15))
    np.testing.assert_array_equal(a.theta, b.theta)


def test_profiling_counts(crv):
    F = W.make_fields("C1")
    w = F.workload
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=1)
    g.set_profiling(True)
    g.step(10)
    ms, n = g.profile(reset=True)
    assert n == 10 and all(x > 0 for x in ms)
    assert g.launches_per_iter > 5


# ------------------------------------------------------------------ backward chain (opt-in path)
@pytest.mark.parametrize("stages", ["1", "2", "4"])
@pytest.mark.parametrize("N,widths,seed", [(64, (2, 256, 256, 256, 256, 256, 1), 11),
                                           (32, (2, 128, 128, 128, 128, 128, 1), 12),
                                           (64, (2, 256, 256, 256, 1), 13)])
def test_backward_chain_vs_oracle(crv, monkeypatch, stages, N, widths, seed):
    """k_tc_bwdc (CRVPINN_BWD_STAGES = S: S hidden GEMMs per launch, Delta handed between stages
    through an L2-resident ring, bias gradients from tensor-core column sums) against the oracle
    at the tensor-mode tolerance, and against the default per-GEMM backward."""
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    rl, rg = oracle.Oracle(N, widths, K, S, f, th).loss_grad()
    monkeypatch.setenv("CRVPINN_BWD_STAGES", stages)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=0)
    loss, grad = g.loss_grad()
    g.close()
    monkeypatch.delenv("CRVPINN_BWD_STAGES")
    tl, tg = TOL[0]
    assert abs(loss - rl) <= tl * abs(rl)
    assert grad_errors(widths, grad, rg).max() <= tg
    d = crv.Crvpinn(N, widths, K, S, f, th, precision=0)
    _, grad_d = d.loss_grad()
    assert grad_errors(widths, grad, grad_d.astype(np.float64)).max() <= 5e-3


# ------------------------------------------------------------------ degenerate and extreme-scale inputs
@pytest.mark.parametrize("prec", PRECS)
def test_zero_problem_is_a_fixed_point(crv, prec):
    """f = 0 and a network whose output layer is zero: u = 0, RES = 0, so LOSS = 0 and every gradient is
    exactly 0 (the zero gradient-scale path: max|gbar| = 0), and Adam leaves theta unchanged bit for bit
    (m = v = 0, so the update is 0 / (0 + eps))."""
    N, widths = 32, (2, 64, 64, 64, 1)
    K, S, _ = W.random_fields(N, 41)
    f = np.zeros_like(K)
    th = W.random_theta(widths, 41)
    off, shape = W.theta_slices(widths)[-2]
    th[off:off + int(np.prod(shape)) + 1] = 0.0               # W_out and b_out
    rl, rg = oracle.Oracle(N, widths, K, S, f, th).loss_grad()
    assert rl == 0.0 and not np.any(rg)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec)
    loss, grad = g.loss_grad()
    assert loss == 0.0 and not np.any(grad)
    assert not np.any(g.eval())
    hist = g.step(5)
    assert not np.any(hist)
    assert np.array_equal(g.theta, th)


@pytest.mark.parametrize("scale", [1e-9, 1e6])
def test_gradient_scale_extremes(crv, scale):
    """The tensor path keeps Delta in fp16 with a power-of-two scale s = 2^(7 - ceil(log2 max|gbar|)):
    gradients many orders of magnitude below fp16's normal range or above its maximum (f scaled by
    1e-9 / 1e6, so RES and gbar scale with it) still match the oracle at the tensor-mode tolerance."""
    N, widths, seed = 64, (2, 128, 128, 128, 1), 42
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    off, shape = W.theta_slices(widths)[-2]
    th[off:off + int(np.prod(shape)) + 1] *= scale            # keep u on the scale of b
    f = (f * scale).astype(np.float32)
    rl, rg = oracle.Oracle(N, widths, K, S, f, th).loss_grad()
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=0)
    loss, grad = g.loss_grad()
    tl, tg = TOL[0]
    assert np.isfinite(loss) and abs(loss - rl) <= tl * abs(rl), (loss, rl)
    assert np.all(np.isfinite(grad))
    assert grad_errors(widths, grad, rg).max() <= tg


@pytest.mark.parametrize("N,widths,scales,seed", [(64, (2, 128, 128, 128, 1), {1: 1e-5, 2: 1e5}, 46),
                                                  (64, (2, 256, 256, 256, 256, 1), {2: 1e-5, 3: 1e5}, 47),
                                                  (32, (2, 64, 64, 64, 1), {1: 1e-5, 2: 1e5}, 48),
                                                  (64, (2, 128, 128, 128, 128, 1), {1: 1e-6, 2: 1e6}, 49)])
def test_hidden_layer_scale_extremes(crv, N, widths, scales, seed):
    """Per-layer exponents of the fp16 weight copies and of Delta, and the 2^14 activation scale
    (DESIGN.md §6): hidden layers scaled by 1e-5 (weights AND biases: the layer runs in tanh's linear
    range, activations ~1e-5, below fp16's normal range without the scale) followed by one scaled by
    1e5 (which undoes it: Delta grows by ~1e5 through one layer). Weights, activations and Delta stay
    in fp16's range; u, the loss and the gradients match the oracle at the tensor-mode tolerances, and
    so they do after an Adam step. (The tanh of the tiny layer must then be accurate RELATIVE to |t|: the next
    layer's gain amplifies absolute errors by 1e5; the forward switches that layer to its
    accurate-tanh path from the gain exponent.)"""
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    sl = W.theta_slices(widths)
    for l, c in scales.items():
        (ow, shw), (ob, shb) = sl[2 * l], sl[2 * l + 1]
        th[ow:ow + int(np.prod(shw))] *= c
        if c < 1:
            th[ob:ob + int(np.prod(shb))] *= c
    th = th.astype(np.float32)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    rl, rg, it = ref.loss_grad(intermediates=True)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=0)
    loss, grad = g.loss_grad()
    u = g.intermediates()["u"]
    tl, tg = TOL[0]
    check_u(0, ref, widths, th, u, it["u"])
    assert np.isfinite(loss) and abs(loss - rl) <= tl * abs(rl), (loss, rl)
    assert np.all(np.isfinite(grad))
    assert grad_errors(widths, grad, rg).max() <= tg, grad_errors(widths, grad, rg)
    # one Adam step moves every tiny weight by ~lr, and the exponents of the next call follow: the GPU
    # at its own new theta against the oracle at that theta. (Not a trajectory comparison: that would
    # only measure the sign-sensitivity of Adam's first step on near-zero gradient components. Nor
    # the gradient there: the step pushes the 1e5 layer into saturation, where 1 - t^2 from an
    # 11-bit t is O(1) wrong in any fp16/TF32-class backward -- DESIGN.md reading R28.)
    g.step(1)
    th1 = g.theta
    rl1 = oracle.Oracle(N, widths, K, S, f, th1).loss_grad()[0]
    l1, g1 = g.loss_grad()
    assert np.isfinite(l1) and abs(l1 - rl1) <= tl * abs(rl1), (l1, rl1)
    assert np.all(np.isfinite(g1))


@pytest.mark.parametrize("N,widths,wscale,seed", [(64, (2,) + (128,) * 10 + (1,), 1.0, 43),
                                                  (64, (2,) + (256,) * 4 + (1,), 3.0, 44),
                                                  (32, (2,) + (64,) * 15 + (1,), 1.0, 45)])
def test_deep_and_saturated_networks(crv, N, widths, wscale, seed):
    """Depth (9 and 14 hidden GEMMs: the fp16 Delta passes through every one of them under one scale)
    and weights 3x the Xavier range (saturated tanh, large pre-activations for the hi/lo split) on the
    tensor path, against the oracle at the tensor-mode tolerance, at theta and after 20 Adam steps."""
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed, scale=wscale)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    rl, rg = ref.loss_grad()
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=0)
    loss, grad = g.loss_grad()
    tl, tg = TOL[0]
    assert abs(loss - rl) <= tl * abs(rl), (loss, rl)
    assert grad_errors(widths, grad, rg).max() <= tg
    hist = g.step(20)
    rh = ref.train(20)
    assert abs(hist[-1] - rh[-1]) <= 0.02 * abs(rh[-1]), (hist[-1], rh[-1])


# ------------------------------------------------------------------ f4: point sharding
@pytest.mark.parametrize("chain", ["0", "1"])
@pytest.mark.parametrize("N,widths,world,seed", [(64, (2, 128, 128, 128, 1), 3, 31),
                                                 (128, (2, 256, 256, 256, 256, 1), 5, 32),
                                                 (64, (2, 64, 64, 64, 1), 2, 33),
                                                 (16, (2, 256, 256, 1), 2, 34)])
def test_point_shards_vs_unsharded_and_oracle(crv, monkeypatch, chain, N, widths, world, seed):
    """`world` shard contexts run one after another on this GPU (no rank waits
    on another), each on its tile range (ragged splits, CTA pairs with odd tile counts); the caller
    does the two exchanges. The summed u is the unsharded u bit for bit (the per-point arithmetic
    does not depend on the tile range), every shard sees the unsharded loss, and the summed gradient
    shares equal the unsharded gradient up to fp32 summation order and the oracle within north_star."""
    monkeypatch.setenv("CRVPINN_BWD_CHAIN", chain)
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    full = crv.Crvpinn(N, widths, K, S, f, th)
    u_ref = full.eval()
    loss_d, grad_d = full.loss_grad()
    full.close()
    shards = [crv.Crvpinn(N, widths, K, S, f, th, shard=(r, world)) for r in range(world)]
    parts = [s.shard_forward() for s in shards]
    support = np.sum([p != 0 for p in parts], axis=0)
    assert support.max() <= 1                                  # disjoint supports
    u = np.sum(parts, axis=0, dtype=np.float32)
    assert np.array_equal(u, u_ref)
    outs = [s.shard_backward(u) for s in shards]
    for loss, _ in outs:
        assert loss == loss_d
    grad = np.sum([g.astype(np.float64) for _, g in outs], axis=0)
    assert grad_errors(widths, grad, grad_d.astype(np.float64)).max() <= 1e-4
    rl, rg = oracle.Oracle(N, widths, K, S, f, th).loss_grad()
    tl, tg = TOL[0]
    assert abs(loss_d - rl) <= tl * abs(rl)
    assert grad_errors(widths, grad, rg).max() <= tg
    with pytest.raises(crv.CrvpinnError) as ei:                # no communicator: the caller exchanges
        shards[0].step(1)
    assert ei.value.code == crv.CRVPINN_EINVAL
    for s in shards:
        s.close()


def test_shard_halves_on_an_unsharded_context(crv):
    """crvpinn_shard_forward / _backward on a world-1 context (no communicator) are the two halves
    of loss_grad: the whole u, then the loss and the whole gradient, bit for bit; theta and the Adam
    state do not move."""
    N, widths, seed = 64, (2, 128, 128, 128, 1), 35
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    g = crv.Crvpinn(N, widths, K, S, f, th)
    loss, grad = g.loss_grad()
    u = g.intermediates()["u"]
    up = g.shard_forward()
    np.testing.assert_array_equal(up, u)
    l2, g2 = g.shard_backward(up)
    assert l2 == loss
    np.testing.assert_array_equal(g2, grad)
    np.testing.assert_array_equal(g.theta, th)
    assert g.adam_state()[2] == 0


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_nccl_world1_matches_unsharded(crv, name):
    """The in-graph exchange (memset of u, NCCL all-reduce of u and of the gradient, captured with the
    100-iteration graph) on a one-rank communicator: the loss history and theta after 100 Adam steps
    equal the unsharded context's bit for bit (a sum over one rank is the identity)."""
    F = W.make_fields(name)
    w = F.workload
    a = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    ha = a.step(100)
    tha = a.theta
    a.close()
    b = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr, shard=(0, 1), nccl_id=crv.nccl_unique_id())
    hb = b.step(100)
    assert np.array_equal(ha, hb)
    assert np.array_equal(tha, b.theta)
    loss, _ = b.loss_grad()
    assert np.isfinite(loss)
    u = b.eval()
    assert np.isfinite(u).all() and np.abs(u).max() > 0
    b.close()


# ------------------------------------------------------------------ f1: gravity term and continuous evaluation
@pytest.mark.parametrize("prec", PRECS)
def test_gravity_term_vs_oracle(crv, prec):
    """A0 with Eq. 23's gravity term (reading R23) against the oracle: the residual of the GPU's own u
    (isolates b), loss and gradients, and again after set_saturation (the term depends on S)."""
    N, widths, seed, Gr = 64, (2, 64, 64, 64, 1), 21, 0.8
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    ref = oracle.Oracle(N, widths, K, S, f, th, gravity=Gr)
    rl, rg, _ = ref.loss_grad(intermediates=True)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec, gravity=Gr)
    loss, grad = g.loss_grad()
    im = g.intermediates()
    r_own = ref.residual(im["u"])
    assert np.max(np.abs(im["res"] - r_own)) <= 1e-5 * np.abs(r_own).max()
    tl, tg = TOL[prec]
    assert abs(loss - rl) <= tl * abs(rl), (loss, rl)
    assert grad_errors(widths, grad, rg).max() <= tg
    rl0 = oracle.Oracle(N, widths, K, S, f, th).loss_grad()[0]
    assert abs(rl - rl0) > 100 * tl * abs(rl)            # the term is not negligible here
    S2 = W.random_fields(N, seed + 1)[1]
    g.set_saturation(S2)
    ref.set_saturation(S2)
    l2, r2 = g.loss_grad(grad=False), ref.loss_grad()[0]
    assert abs(l2 - r2) <= tl * abs(r2), (l2, r2)


@pytest.mark.parametrize("prec", PRECS)
def test_eval_points_vs_oracle(crv, prec):
    """crvpinn_eval_points (continuous evaluation for the IGA projection) against
    the oracle at random points (ragged count, inside and outside the unit square), exact zeros on the
    boundary, bitwise agreement with the lattice forward at the lattice nodes, more points than the
    lattice holds, n = 0 and a non-finite coordinate."""
    N, widths, seed = 32, (2, 128, 128, 128, 1), 22
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    rng = np.random.default_rng(seed)
    xy = np.concatenate([rng.uniform(0, 1, (1000, 2)), rng.uniform(-0.25, 1.25, (77, 2))]).astype(np.float32)
    p, pr = g.eval_points(xy), ref.eval_points(xy)
    tol = (1e-5 if prec == 1 else 2e-3) * np.abs(pr).max()
    assert np.max(np.abs(p - pr)) <= tol
    t = np.linspace(0, 1, 37, dtype=np.float32)
    edge = np.concatenate([np.stack([np.zeros_like(t), t], 1), np.stack([t, np.ones_like(t)], 1)])
    assert np.all(g.eval_points(edge) == 0.0)
    i, j = np.meshgrid(np.arange(N + 1), np.arange(N + 1))
    lat = np.stack([i.reshape(-1) / N, j.reshape(-1) / N], 1).astype(np.float32)
    np.testing.assert_array_equal(g.eval_points(lat), g.eval())
    big = rng.uniform(0, 1, (N * N + 300, 2)).astype(np.float32)
    pb = g.eval_points(big)
    idx = rng.choice(big.shape[0], 200, replace=False)
    assert np.max(np.abs(pb[idx] - ref.eval_points(big[idx]))) <= (1e-5 if prec == 1 else 2e-3) * np.abs(pr).max()
    assert g.eval_points(np.zeros((0, 2), np.float32)).shape == (0,)
    bad = xy[:5].copy()
    bad[3, 1] = np.nan
    with pytest.raises(crv.CrvpinnError) as e:
        g.eval_points(bad)
    assert e.value.code == crv.CRVPINN_EDOMAIN


@pytest.mark.parametrize("prec", PRECS)
def test_eval_points_chunk_pipeline(crv, prec):
    """crvpinn_eval_points streams its points through two 2^18-point chunk buffers (pinned staging, copy
    stream): 2 chunks + a ragged tail give the same values bit for bit as evaluating every piece on its
    own (the per-point arithmetic does not depend on the chunk), sampled points match the oracle, the
    output of a non-finite call is untouched (nothing is written), and training in between is seen."""
    N, widths, seed = 32, (2, 128, 128, 128, 1), 23
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    rng = np.random.default_rng(seed)
    C = 1 << 18
    n = 2 * C + 12345
    xy = rng.uniform(-0.1, 1.1, (n, 2)).astype(np.float32)
    p = g.eval_points(xy)
    pieces = np.concatenate([g.eval_points(xy[a:b]) for a, b in ((0, 1000), (1000, C + 7), (C + 7, n))])
    np.testing.assert_array_equal(p, pieces)
    idx = np.concatenate([rng.choice(n, 200, replace=False), [0, C - 1, C, 2 * C - 1, 2 * C, n - 1]])
    pr = ref.eval_points(xy[idx])
    assert np.max(np.abs(p[idx] - pr)) <= (1e-5 if prec == 1 else 2e-3) * np.abs(pr).max()
    out = np.full(n, 7.0, np.float32)
    bad = xy.copy()
    bad[C + 5, 0] = np.inf
    rc = crv.load().crvpinn_eval_points(g._h, n, crv._fp(bad), crv._fp(out))   # the raw call: out is ours
    assert rc == crv.CRVPINN_EDOMAIN
    assert np.all(out == 7.0)
    g.step(3)
    p2 = g.eval_points(xy[:5000])
    np.testing.assert_array_equal(p2, g.eval_points(xy[:5000]))
    assert not np.array_equal(p2, p[:5000])


# ------------------------------------------------------------------ f2: the discrete system by Gram-preconditioned CG
@pytest.mark.parametrize("N,seed,Gr", [(32, 31, 0.0), (64, 32, 0.5), (128, 33, 0.0)])
def test_direct_solve_vs_oracle(crv, N, seed, Gr):
    """crvpinn_direct_solve against the oracle's band-LU solve of A(alpha) u = b:
    the reported true residual (fp64 iterate) meets rtol, the oracle's residual of the returned fp32 u
    is that plus fp32 rounding, and
    the solution error is within the conditioning bound kappa * rtol (kappa <= max alpha / min alpha
    times the Gram spectral bound, P6)."""
    widths = (2, 32, 32, 1)
    K, S, f = W.random_fields(N, seed)
    g = crv.Crvpinn(N, widths, K, S, f, precision=1, gravity=Gr)
    ref = oracle.Oracle(N, widths, K, S, f, gravity=Gr)
    rtol = 1e-6
    u, it, rel = g.direct_solve(rtol=rtol, max_iter=5000)
    assert rel <= 2 * rtol and it < 5000, (it, rel)
    U = u.reshape(N + 1, N + 1)
    assert np.all(U[0] == 0) and np.all(U[-1] == 0) and np.all(U[:, 0] == 0) and np.all(U[:, -1] == 0)
    b = -ref.residual(np.zeros((N + 1) ** 2))
    # rel is the residual of the fp64 iterate; the returned u is its fp32 rounding
    rel_o = np.linalg.norm(ref.residual(u.astype(np.float64))) / np.linalg.norm(b)
    assert rel_o <= rel + 5e-5, (rel_o, rel)
    ustar = ref.direct_solve()
    a = ref.alpha().reshape(N + 1, N + 1)[:N, :N]
    kappa = a.max() / a.min()
    err = np.linalg.norm(u - ustar) / np.linalg.norm(ustar)
    assert err <= 10 * kappa * rtol, (err, kappa)


def test_direct_solve_edges(crv):
    F = W.make_fields("C1")
    w = F.workload
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=0)
    th = g.theta.copy()
    with pytest.raises(crv.CrvpinnError):
        g.direct_solve(rtol=0.0)
    u, it, rel = g.direct_solve(rtol=1e-5, max_iter=1)
    assert it == 1 and rel > 0
    u, it, rel = g.direct_solve(rtol=1e-6)
    assert rel <= 2e-6
    # C1: alpha = 1, f = 2 pi^2 sin sin => u* = c_h sin sin exactly (P4), c_h = (pi h/2)^2 / sin^2(pi h/2)
    N = w.N
    i, j = np.meshgrid(np.arange(N + 1), np.arange(N + 1))
    c_h = (np.pi / (2 * N)) ** 2 / np.sin(np.pi / (2 * N)) ** 2
    ustar = c_h * np.sin(np.pi * i / N) * np.sin(np.pi * j / N)
    assert np.max(np.abs(u - ustar.reshape(-1))) <= 1e-5 * ustar.max()
    np.testing.assert_array_equal(g.theta, th)       # the solve leaves the network alone


# ------------------------------------------------------------------ f3: IGA-ADS saturation step
def _iga_pair(crv, ne, r):
    return crv.Iga(ne, r), oracle.IgaOracle(ne, r)


def _mass_dense(o):
    """The oracle's 1-D mass matrix as a dense array (banded storage [nb][r+1]: M_{j,j+d})."""
    M = np.asarray(o.mass_1d())
    nb, r = o.nb, o.r
    if M.ndim == 2 and M.shape == (nb, nb):
        return M
    B = M.reshape(nb, r + 1)
    F = np.zeros((nb, nb))
    for j in range(nb):
        for d in range(r + 1):
            if j + d < nb:
                F[j, j + d] = F[j + d, j] = B[j, d]
    return F


@pytest.mark.parametrize("ne,r", [(8, 1), (16, 2), (37, 2), (20, 3), (100, 3), (64, 4), (70, 5), (40, 6)])
def test_iga_projection_and_eval_vs_oracle(crv, ne, r):
    """crvpinn_iga_project / _eval against the fp64 oracle: quadrature points,
    projected coefficients of a smooth function, exact reproduction of x^2 + y^2 (degree >= 2), and
    values/gradients at random points."""
    g, o = _iga_pair(crv, ne, r)
    assert g.nb == o.nb == ne + r
    q = g.quad_points()
    np.testing.assert_allclose(q, o.quad_points(), atol=2e-7)
    f = (np.sin(3 * q[:, 0]) * np.cos(2 * q[:, 1]) + q[:, 1]).astype(np.float32)
    C, Co = g.project(f), o.project(f.astype(np.float64))
    # the fp32 load vector's rounding is amplified by the 2-D mass matrix's condition number
    # (1e2 at degree 2, 7e2 at 3, 5e3 at 4, 3e4 at 5, 2e5 at 6; DESIGN.md §9 f3): 5e-9 kappa, 12x
    # below the worst case 2^-24 kappa, floored at 1e-5
    M1 = _mass_dense(o)
    tol = max(1e-5, 5e-9 * np.linalg.cond(M1) ** 2)
    assert np.max(np.abs(C - Co)) <= tol * np.abs(Co).max()
    rng = np.random.default_rng(ne)
    pts = rng.uniform(0, 1, (500, 2)).astype(np.float32)
    v, gr = g.eval(C, pts, grad=True)
    vo, gro = o.eval(Co, pts, grad=True)
    assert np.max(np.abs(v - vo)) <= 1e-5 * np.abs(vo).max()
    assert np.max(np.abs(gr - gro)) <= 1e-4 * np.abs(gro).max()
    if r >= 2:
        C2 = g.project((q[:, 0] ** 2 + q[:, 1] ** 2).astype(np.float32))
        np.testing.assert_allclose(g.eval(C2, pts), pts[:, 0] ** 2 + pts[:, 1] ** 2, atol=2e-6)


@pytest.mark.parametrize("ne,r,Gr", [(16, 2, 0.0), (48, 2, 1.5), (33, 1, 0.7), (100, 3, 0.4), (64, 4, 1.0),
                                     (70, 5, 0.0), (40, 6, 0.8)])
def test_iga_saturation_step_vs_oracle(crv, ne, r, Gr):
    """One explicit step of Eq. 10 (readings R24-R26) on the GPU against the oracle, with
    heterogeneous K, a source patch, a non-trivial pressure and gravity."""
    g, o = _iga_pair(crv, ne, r)
    q = g.quad_points().astype(np.float64)
    S = o.project(np.exp(-((q[:, 0] - 0.5) ** 2 + (q[:, 1] - 0.45) ** 2) / 0.02))
    S[0, :] = S[-1, :] = S[:, 0] = S[:, -1] = 0.0
    P = o.project(np.cos(2 * q[:, 0]) * q[:, 1] - Gr * q[:, 1])
    rng = np.random.default_rng(ne + r)
    K = np.exp(rng.standard_normal((ne, ne)) * 0.5)
    src = np.zeros((ne, ne))
    src[ne // 3:ne // 2, ne // 3:ne // 2] = 1.0
    args = dict(tau=0.02, phi=0.3, gravity=Gr)
    S1 = g.saturation_step(S.astype(np.float32), P.astype(np.float32), K.astype(np.float32),
                           src.astype(np.float32), **args)
    S1o = o.saturation_step(S.astype(np.float32).astype(np.float64), P.astype(np.float32).astype(np.float64),
                            K.astype(np.float32).astype(np.float64), src, **args)
    assert np.max(np.abs(S1 - S1o)) <= 2e-5 * np.abs(S1o).max()
    assert np.all(S1[0, :] == 0) and np.all(S1[-1, :] == 0) and np.all(S1[:, 0] == 0) and np.all(S1[:, -1] == 0)
    assert g.last_ms > 0


def test_iga_buoyancy_at_size_and_hybrid_loop(crv):
    """At ne = 256 (the paper's scale of 100x100 IGA elements and above) the gas blob rises under a
    hydrostatic water pressure (property of any size, reading R24), and one hybrid round trip runs
    end to end: CRVPINN pressure at the Gauss points (f1) -> L2 projection -> saturation step ->
    saturation at the collocation lattice -> crvpinn_set_saturation -> 100 Adam iterations."""
    g = crv.Iga(256, 2)
    q = g.quad_points()
    S = g.project(np.exp(-((q[:, 0] - 0.5) ** 2 + (q[:, 1] - 0.4) ** 2) / 0.01).astype(np.float32))
    S[0, :] = S[-1, :] = S[:, 0] = S[:, -1] = 0.0
    Gr = 2.0
    P = g.project((-Gr * q[:, 1]).astype(np.float32))
    K = np.ones((256, 256), np.float32)
    S1 = g.saturation_step(S, P, K, np.zeros_like(K), tau=1e-3, gravity=Gr)
    grid = np.stack(np.meshgrid(np.linspace(0, 1, 257), np.linspace(0, 1, 257)), -1).reshape(-1, 2).astype(np.float32)
    s0, s1 = g.eval(S, grid).astype(np.float64), g.eval(S1, grid).astype(np.float64)
    assert (s1 * grid[:, 1]).sum() / s1.sum() > (s0 * grid[:, 1]).sum() / s0.sum()
    F = W.make_fields("C3")
    w = F.workload
    c = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=0, lr=w.lr)
    gi = crv.Iga(64, 2)
    p_q = c.eval_points(gi.quad_points())
    P = gi.project(p_q)
    S0 = gi.project(np.zeros(gi.nq, np.float32))
    Kq = np.ones((64, 64), np.float32)
    src = np.zeros((64, 64), np.float32)
    src[30:34, 30:34] = 5.0
    S1 = gi.saturation_step(S0, P, Kq, src, tau=0.05)
    N = w.N
    i, j = np.meshgrid(np.arange(N + 1), np.arange(N + 1))
    lat = np.stack([i.reshape(-1) / N, j.reshape(-1) / N], 1).astype(np.float32)
    S_lat = np.clip(gi.eval(S1, lat), 0, 1)
    c.set_saturation(S_lat)
    hist = c.step(100)
    assert np.all(np.isfinite(hist)) and S_lat.max() > 0


def test_iga_edges(crv):
    with pytest.raises(crv.CrvpinnError):
        crv.Iga(0, 2)
    with pytest.raises(crv.CrvpinnError):
        crv.Iga(8, 7)
    g = crv.Iga(8, 2)
    z = np.zeros((g.nb, g.nb), np.float32)
    e = np.zeros((8, 8), np.float32)
    with pytest.raises(crv.CrvpinnError):
        g.saturation_step(z, z, e, e, tau=-1.0)
    assert g.eval(z, np.zeros((0, 2))).shape == (0,)


# ------------------------------------------------------------------ maximum size (N = 2048)
def test_maximum_grid_properties(crv):
    """N = 2048 (the largest grid the ABI accepts; 4.2 M MLP points, 21 GB of fp16 activations) with
    the C5 network: the oracle cannot run the whole iteration at this size, so each step is checked
    where it can be computed one by one -- u at 1000 sampled nodes against the oracle's evaluation
    there, RES against the oracle's stencil on the GPU's own u, q through G q = RES (oracle stencil
    form of G), dLOSS/du against the oracle's adjoint of the GPU's q -- plus exact boundary zeros."""
    N, widths = 2048, (2, 256, 256, 256, 256, 256, 1)
    K, S, f = W.random_fields(N, 2048)
    th = W.random_theta(widths, 2048)
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=0)
    loss, grad = g.loss_grad()
    assert np.isfinite(loss) and loss > 0 and np.all(np.isfinite(grad))
    im = g.intermediates()
    U = im["u"].reshape(N + 1, N + 1)
    assert np.all(U[0] == 0) and np.all(U[-1] == 0) and np.all(U[:, 0] == 0) and np.all(U[:, -1] == 0)
    ref = oracle.Oracle(N, widths, K, S, f, th, factor_gram=False)
    rng = np.random.default_rng(7)
    idx = rng.choice((N + 1) ** 2, 1000, replace=False)
    xy = np.stack([(idx % (N + 1)) / N, (idx // (N + 1)) / N], 1)
    u_ref = ref.eval_points(xy)
    assert np.max(np.abs(im["u"][idx] - u_ref)) <= 2e-3 * np.abs(u_ref).max()
    r_own = ref.residual(im["u"])
    assert np.max(np.abs(im["res"] - r_own)) <= 1e-5 * np.abs(r_own).max()
    gq = ref.gram_matvec(im["q"].astype(np.float64))
    assert np.linalg.norm(gq - im["res"]) <= 1e-3 * np.linalg.norm(im["res"])
    gu_own = ref.residual_adjoint(2.0 * im["q"].astype(np.float64))
    mask = np.zeros((N + 1, N + 1))
    mask[1:-1, 1:-1] = 1
    gu_own *= mask.reshape(-1)
    assert np.max(np.abs(im["gu"] - gu_own)) <= 1e-5 * np.abs(gu_own).max()
    g.close()
