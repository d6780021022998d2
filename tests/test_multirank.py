"""World-size-2 tests of the point-sharded path on CPU
over torch.distributed `gloo`: the shard split, the communicator-id exchange, and the sharded
decomposition of one iteration -- each rank's forward on its rows, an all-reduce of u, the
replicated stencil / Gram / adjoint, each rank's backward on its rows, an all-reduce of the
gradient -- carried out with the fp64 oracle as the per-rank compute, so that the exchange
pattern the CUDA path issues (crvpinn.cu: launch_iteration) is checked end to end without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2604_20731_b200 as crv

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def _run(fn, world=WORLD):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


# ---------------------------------------------------------------- shard split
def _tiles(rank, world):
    res = {}
    for N in (16, 32, 64, 128, 256, 512, 1024, 2048):
        t0, nt = crv.shard_tiles(N, rank, world)
        got = [None] * world
        dist.all_gather_object(got, (t0, nt))
        res[N] = got
    return res


def test_shard_tiles_partition_gloo():
    res = _run(_tiles)
    assert res[0] == res[1]
    for N, parts in res[0].items():
        T = N * N // 128
        cover = []
        for t0, nt in parts:
            assert nt >= 1
            cover.extend(range(t0, t0 + nt))
        assert cover == list(range(T)), N                      # disjoint, ordered, complete
        sizes = [nt for _, nt in parts]
        assert max(sizes) - min(sizes) <= 1


def test_shard_tiles_host_rules():
    for N in (16, 64, 512):
        T = N * N // 128
        for w in sorted({1, 2, 3, 7, T} & set(range(1, T + 1))):
            parts = [crv.shard_tiles(N, r, w) for r in range(w)]
            assert sum(nt for _, nt in parts) == T
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(w - 1))
    for bad in [(64, 0, 0), (64, 2, 2), (64, -1, 2), (64, 0, 33), (48, 0, 1)]:
        with pytest.raises(crv.CrvpinnError):
            crv.shard_tiles(*bad)


def test_sharded_create_rejected_before_device():
    N = 32
    nn = (N + 1) ** 2
    for shard in [(2, 2), (0, 9), (-1, 2)]:
        with pytest.raises(crv.CrvpinnError) as ei:
            crv.Crvpinn(N, (2, 32, 1), np.ones(nn), np.zeros(nn), np.zeros(nn), shard=shard)
        assert ei.value.code == crv.CRVPINN_EINVAL
    with pytest.raises(crv.CrvpinnError) as ei:   # the fp32 SIMT path does not shard
        crv.Crvpinn(N, (2, 32, 1), np.ones(nn), np.zeros(nn), np.zeros(nn), shard=(0, 2),
                    precision=crv.PREC_FP32)
    assert ei.value.code == crv.CRVPINN_EINVAL and "tensor" in str(ei.value)


# ---------------------------------------------------------------- communicator id
def _share_id(rank, world):
    return crv.share_nccl_id()


def test_nccl_id_shared_gloo():
    ids = _run(_share_id)
    assert len(ids[0]) == 128 and ids[0] == ids[1] and any(ids[0])


# ---------------------------------------------------------------- sharded iteration (oracle compute)
def _sharded_oracle(rank, world):
    import torch
    import oracle
    import workloads as W
    F = W.make_fields("C2")
    w = F.workload
    orc = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0)
    N = w.N
    # rows of the MLP point set, split like the tiles (whole rows here: N = 64 -> 2 rows per tile)
    t0, nt = crv.shard_tiles(N, rank, world)
    j0, j1 = 1 + t0 * 128 // N, 1 + (t0 + nt) * 128 // N
    u_part = orc.forward_rows(j0, j1)
    u = torch.from_numpy(u_part.copy())
    dist.all_reduce(u)                                         # exchange 1: u
    loss, _, q = orc.loss_u(u.numpy())                         # replicated A2-A5
    gu = orc.residual_adjoint(2.0 * q)
    g = torch.from_numpy(orc.grad_rows(gu, j0, j1))
    dist.all_reduce(g)                                         # exchange 2: dLOSS/dtheta
    return loss, g.numpy(), u.numpy(), (j0, j1)


def test_point_sharded_iteration_matches_unsharded_gloo():
    import oracle
    import workloads as W
    res = _run(_sharded_oracle)
    F = W.make_fields("C2")
    w = F.workload
    orc = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0)
    loss_ref, g_ref, inter = orc.loss_grad(intermediates=True)
    rows = sorted(r[3] for r in res)
    assert rows[0][0] == 1 and rows[-1][1] == w.N + 1 and rows[0][1] == rows[1][0]
    for loss, g, u, _ in res:
        np.testing.assert_allclose(u, inter["u"], rtol=0, atol=0)           # disjoint supports: exact
        assert abs(loss - loss_ref) <= 1e-14 * abs(loss_ref)
        assert np.linalg.norm(g - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
