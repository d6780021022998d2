"""Long oracle runs for the multi-step parity fixtures (tests/golden/), oracle only (fp64).

Calls only oracle/ and the seeded input generators (workloads/); nothing here touches the CUDA
path. Each sub-command writes one .npz under tests/golden/.

  c4sched                 C4's full schedule (§6 step 7; BASELINE.json configs[3]):
                          10 time steps x 100 Adam iterations, warm-started weights and Adam state,
                          S advanced between steps (S_steps[k] for step k) -> C4_sched10x100.npz
  c5sched [steps] [--resume]  the same for C5 (configs[4]), the first [steps] time steps (the fixture is
                          rewritten after every step: steps_done) -> C5_sched.npz
  c3 <seed> <iters>       C3's pretraining + updates with fixed S (configs[2]):
                          <iters> Adam iterations from theta0 (seed 0) or from theta0 moved by one fp32
                          ulp per entry (seed > 0, the recipe of scripts/c3_sensitivity.py)
                          -> C3_run<iters>_s<seed>.npz
  c3model <seed> <iters> [--bits B]
                          the same iteration in the B-bit precision class (default 11: fp16 / TF32;
                          24: fp32) (oracle/precision_model.py, reading R28)
                          -> C3_model<B>_run<iters>_s<seed>.npz
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def ulp_perturbed(theta0, seed):
    t0 = np.asarray(theta0, dtype=np.float32)
    if seed == 0:
        return t0
    rng = np.random.default_rng(seed)
    return np.nextafter(t0, np.where(rng.random(t0.shape) < 0.5, -np.inf, np.inf).astype(np.float32))


def sched(name="C4", max_steps=None, resume=False):
    """name's schedule (C4: all 10 steps -> C4_sched10x100.npz; C5: the first max_steps of its 10,
    rewritten after every step so a partial run is usable -> C5_sched.npz with steps_done, plus the
    fp64 state after the last step (theta, m, v, t) so that `resume` continues the run exactly).
    S_steps[k] is the saturation of time step k; a workload with one S (C5) keeps it."""
    F = W.make_fields(name)
    w = F.workload
    n = w.n_steps if max_steps is None else min(max_steps, w.n_steps)
    t = time.time()
    o = oracle.Oracle(w.N, w.widths, F.K, F.S_steps[0], F.f, F.theta0, lr=w.lr)
    hist = np.zeros((n, w.n_adam))
    step_end = np.zeros(n)
    thetas = {}
    fname = "C4_sched10x100.npz" if name == "C4" else f"{name}_sched.npz"
    k0 = 0
    if resume:
        z = np.load(os.path.join(OUT, fname))
        k0 = int(z["steps_done"])
        hist[:k0], step_end[:k0] = z["hist"][:k0], z["step_end"][:k0]
        thetas = {key: z[key] for key in z.files if key.startswith("theta_step")}
        o.theta = z["state_theta"]
        o.set_adam_state(z["state_m"], z["state_v"], int(z["state_t"]))
        if k0 < len(F.S_steps) and k0 > 0:
            o.set_saturation(F.S_steps[k0 - 1])
    for k in range(k0, n):
        if 0 < k < len(F.S_steps):
            o.set_saturation(F.S_steps[k])
        hist[k] = o.train(w.n_adam)
        step_end[k] = o.loss_grad()[0]      # LOSS(theta after step k) on the step's S
        if k in (0, w.n_steps - 1):
            thetas[f"theta_step{k + 1}"] = o.theta.astype(np.float32)
        print(f"{name} step {k + 1}: {hist[k, 0]:.6e} -> {hist[k, -1]:.6e} end {step_end[k]:.6e} "
              f"({time.time() - t:.0f}s)", flush=True)
        if name != "C4" or k == n - 1:
            m, v, tt = o.adam_state()
            np.savez_compressed(os.path.join(OUT, fname), hist=hist[:k + 1], step_end=step_end[:k + 1],
                                steps_done=k + 1, threads=oracle.max_threads(), state_theta=o.theta,
                                state_m=m, state_v=v, state_t=tt, **thetas)


def c3model(seed, iters, bits=11):
    from oracle.precision_model import PrecisionModel
    F = W.make_fields("C3")
    w = F.workload
    t = time.time()
    pm = PrecisionModel(w.N, w.widths, F.K, F.S, F.f, ulp_perturbed(F.theta0, seed), lr=w.lr, bits=bits)
    chunks = []
    for i0 in range(0, iters, 500):
        chunks.append(pm.train(min(500, iters - i0)))
        print(f"C3 model{bits} s{seed}: it {i0 + len(chunks[-1])} loss {chunks[-1][-1]:.6e} ({time.time() - t:.0f}s)",
              flush=True)
    name = f"C3_model{bits}_run{iters}_s{seed}.npz"
    np.savez_compressed(os.path.join(OUT, name), hist=np.concatenate(chunks), seed=seed, bits=bits)
    print(f"wrote {name} ({time.time() - t:.0f}s)", flush=True)


def c3(seed, iters, noise):
    F = W.make_fields("C3")
    w = F.workload
    t = time.time()
    o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, ulp_perturbed(F.theta0, seed), lr=w.lr)
    if noise > 0:
        rng = np.random.Generator(np.random.PCG64(1000 + seed))
        hist = np.zeros(iters)
        for i in range(iters):
            loss, g = o.loss_grad()
            hist[i] = loss
            xi = rng.standard_normal(g.shape)
            o.adam_step(g + noise * (np.linalg.norm(g) / np.sqrt(g.size)) * xi)
            if (i + 1) % 500 == 0:
                print(f"C3 s{seed} noise {noise:g}: it {i + 1} loss {loss:.6e} ({time.time() - t:.0f}s)", flush=True)
        name = f"C3_run{iters}_s{seed}_noise{noise:g}.npz"
    else:
        chunks = []
        for i0 in range(0, iters, 500):
            chunks.append(o.train(min(500, iters - i0)))
            print(f"C3 s{seed}: it {i0 + len(chunks[-1])} loss {chunks[-1][-1]:.6e} ({time.time() - t:.0f}s)",
                  flush=True)
        hist = np.concatenate(chunks)
        name = f"C3_run{iters}_s{seed}.npz"
    np.savez_compressed(os.path.join(OUT, name), hist=hist, final_loss=np.float64(o.loss_grad()[0]),
                        theta=o.theta.astype(np.float32), seed=seed, noise=noise, threads=oracle.max_threads())
    print(f"wrote {name} ({time.time() - t:.0f}s)", flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "c4sched":
        sched("C4")
    elif cmd == "c5sched":
        sched("C5", int(sys.argv[2]) if len(sys.argv) > 2 else None, resume="--resume" in sys.argv)
    elif cmd == "c3model":
        bits = int(sys.argv[sys.argv.index("--bits") + 1]) if "--bits" in sys.argv else 11
        c3model(int(sys.argv[2]), int(sys.argv[3]), bits)
    elif cmd == "c3":
        noise = float(sys.argv[sys.argv.index("--noise") + 1]) if "--noise" in sys.argv else 0.0
        c3(int(sys.argv[2]), int(sys.argv[3]), noise)
    else:
        raise SystemExit(__doc__)
