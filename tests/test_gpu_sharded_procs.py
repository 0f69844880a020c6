"""Time-sharded path with REAL ranks: world = 2 and 3 processes,
each driving libpssgp.so's shard phases (sharded.DeviceShard) on cuda:0, exchanging the
aggregate blobs over gloo through host memory (the NCCL all_gather of bench.py, with a CPU hop).
No kernel of one rank waits on another rank: every exchange happens between launches, on the host.
The result of every rank must equal the unsharded posterior to 1e-11 (the grouping of the scan is
arbitrary), and every rank must report the same total NLL (the library's
fixed-order sum of the gathered partials).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind):
    if kind == "matern52":
        return synth.random_problem(23, 200_003, kind="matern52", p_missing=0.2, ties=3)
    # wide path (d = 6, uniform dt)
    n, dt = 50_001, synth.H_FINE * 8
    t = np.arange(n, dtype=np.float64) * dt
    rng = np.random.default_rng(4)
    mask = (rng.random(n) >= 0.1).astype(np.uint8)
    y = synth.sinusoid(t) + 0.1 * rng.standard_normal(n)
    y[mask == 0] = np.nan
    return synth.Workload("rbf6", [synth.Component("rbf", 1.0, 0.5, order=6)], 0.01, t, y, mask, uniform_dt=dt)


def _gloo_exchange(x):
    """all_gather of a device tensor through host memory (gloo), stacked [world, ...] on the device."""
    torch.cuda.synchronize()
    h = x.detach().cpu()
    parts = [torch.empty_like(h) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, h)
    return torch.stack(parts).to(x.device)


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2102_09964_b200 as P
        from paper_2102_09964_b200 import sharded
        w = _problem(kind)
        k0, n = sharded.split(w.N, world)[rank]
        m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
        tt, yy, mm = sharded.chunk_inputs(w.t, w.y, w.mask, k0, n, "cuda:0")
        shard = sharded.DeviceShard(m, tt, yy, mm, k0, n, w.N, rank, world)
        mean, var, nll = sharded.sharded_posterior(shard, _gloo_exchange, rank, world)
        m.check()
        q.put((rank, mean.cpu().numpy(), var.cpu().numpy(), float(nll.cpu()[0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["matern52", "rbf6"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ranks_match_unsharded(cuda_device, world, kind):
    import paper_2102_09964_b200 as P
    w = _problem(kind)
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
    t, y, mk = (torch.from_numpy(a).to(cuda_device) for a in (w.t, w.y, w.mask))
    ref_mean, ref_var, ref_nll = (x.cpu().numpy() for x in m.posterior(t, y, mk))
    m.check()
    ref_nll = float(ref_nll[0])

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    mean = np.concatenate([r[1] for r in res])
    var = np.concatenate([r[2] for r in res])
    nlls = [r[3] for r in res]
    assert all(v == nlls[0] for v in nlls)                 # the same fixed-order total on every rank
    assert np.max(np.abs(mean - ref_mean)) / np.max(np.abs(ref_mean)) < 1e-11
    assert np.max(np.abs(var - ref_var) / ref_var) < 1e-11
    assert abs(nlls[0] - ref_nll) < 1e-11 * abs(ref_nll)
