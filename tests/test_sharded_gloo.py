"""Multi-process (world_size 2 and 3, gloo on CPU) test of the time-sharded
protocol in paper_2102_09964_b200/sharded.py: the exchange order (filter
aggregates of ranks < g, smoother aggregates of ranks > g), the one-point
halo of t, the global first / terminal elements and the NLL partials carried
in the smoother blobs.

The per-rank backend here is a MOCK built from the oracle's element algebra
(oracle/elements.py) — it exercises the protocol and the
collectives, not the CUDA kernels (those are covered by the GPU virtual-sharding
test).  The result must equal the sequential oracle (Props. 1, 2).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from oracle import elements as el
from oracle import ssm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleShard:
    """numpy backend for one rank (full matrices, oracle algebra)."""

    def __init__(self, m, r, t, y, mask, k0, n, N):
        self.m, self.r, self.k0, self.n, self.N = m, r, k0, n, N
        self.t, self.y, self.mask = t, y, mask          # global arrays (halo read explicitly)
        d = m.n
        self.d = d
        F = {}; Q = {}
        for k in range(max(k0, 1), min(k0 + n + 1, N)):  # transitions into k, incl. the halo step k0+n
            F[k], Q[k] = oracle.discretize(m, t[k] - t[k - 1])
        self.F, self.Q = F, Q

    def _flat(self, tup):
        return torch.from_numpy(np.concatenate([np.ravel(x) for x in tup]))

    def _unflat_f(self, v):
        d = self.d; v = v.numpy(); o = 0
        A = v[o:o + d * d].reshape(d, d); o += d * d
        b = v[o:o + d]; o += d
        C = v[o:o + d * d].reshape(d, d); o += d * d
        eta = v[o:o + d]; o += d
        J = v[o:o + d * d].reshape(d, d)
        return (A, b, C, eta, J)

    def _unflat_s(self, v):
        d = self.d; v = v.numpy()
        return (v[:d * d].reshape(d, d), v[d * d:d * d + d], v[d * d + d:].reshape(d, d))

    def _elements(self):
        k0, n = self.k0, self.n
        Fl = [self.F.get(k) for k in range(k0, k0 + n)]
        Ql = [self.Q.get(k) for k in range(k0, k0 + n)]
        if k0 > 0:
            # filter_elements treats list index 0 as the global first step; shift by a dummy
            Fl = [None] + Fl; Ql = [None] + Ql
            ys = np.concatenate([[0.0], self.y[k0:k0 + n]]); ms = np.concatenate([[0], self.mask[k0:k0 + n]])
            return el.filter_elements(Fl, Ql, self.m.H, self.m.Pinf, self.r, ys, ms)[1:]
        return el.filter_elements(Fl, Ql, self.m.H, self.m.Pinf, self.r, self.y[:n], self.mask[:n])

    def filter_reduce(self):
        self.fe = self._elements()
        agg = self.fe[0]
        for e in self.fe[1:]:
            agg = el.filter_combine(agg, e)
        return self._flat(agg)

    def filter_apply(self, all_fa):
        rank = self.rank
        carry = None
        for g in range(rank):
            a = self._unflat_f(all_fa[g])
            carry = a if carry is None else el.filter_combine(carry, a)
        pref = []
        acc = carry
        for e in self.fe:
            acc = e if acc is None else el.filter_combine(acc, e)
            pref.append(acc)
        self.xf = np.array([p_[1] for p_ in pref]); self.Pf = np.array([p_[2] for p_ in pref])
        # NLL partial from the predictive decomposition
        nll = 0.0
        H = self.m.H
        for i in range(self.n):
            k = self.k0 + i
            if not self.mask[k]:
                continue
            if k == 0:
                xm, Pm = np.zeros(self.d), self.m.Pinf
            else:
                xp = self.xf[i - 1] if i > 0 else carry[1]
                Pp = self.Pf[i - 1] if i > 0 else carry[2]
                xm, Pm = self.F[k] @ xp, self.F[k] @ Pp @ self.F[k].T + self.Q[k]
            S = H @ Pm @ H + self.r
            v = self.y[k] - H @ xm
            nll += 0.5 * (np.log(2 * np.pi * S) + v * v / S)
        # smoother aggregate of the chunk (terminal on the last rank)
        Fn = {k - self.k0: self.F[k] for k in self.F}
        Qn = {k - self.k0: self.Q[k] for k in self.Q}
        se = []
        for i in range(self.n):
            k = self.k0 + i
            if k == self.N - 1:
                se.append((np.zeros((self.d, self.d)), self.xf[i], self.Pf[i]))
            else:
                Fk, Qk = Fn[i + 1], Qn[i + 1]
                Pm = Fk @ self.Pf[i] @ Fk.T + Qk
                E = np.linalg.solve(Pm, Fk @ self.Pf[i]).T
                se.append((E, self.xf[i] - E @ Fk @ self.xf[i], self.Pf[i] - E @ Fk @ self.Pf[i]))
        self.se = se
        agg = se[0]
        for e in se[1:]:
            agg = el.smoother_combine(agg, e)
        # one blob: the smoother aggregate followed by the NLL partial (as the library's)
        return torch.cat([self._flat(agg), torch.tensor([nll], dtype=torch.float64)])

    def smoother_apply(self, all_sb):
        world = all_sb.shape[0]
        carry = None
        for g in range(world - 1, self.rank, -1):
            a = self._unflat_s(all_sb[g][:-1])
            carry = a if carry is None else el.smoother_combine(a, carry)
        acc = carry
        means = np.empty(self.n); vars_ = np.empty(self.n)
        for i in range(self.n - 1, -1, -1):
            acc = self.se[i] if acc is None else el.smoother_combine(self.se[i], acc)
            means[i] = self.m.H @ acc[1]
            vars_[i] = self.m.H @ acc[2] @ self.m.H
        nll = 0.0
        for g in range(world):                       # fixed-order sum of the gathered partials
            nll += float(all_sb[g][-1])
        return torch.from_numpy(means), torch.from_numpy(vars_), torch.tensor([nll], dtype=torch.float64)


def _worker(rank, world, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_09964_b200 import sharded
        w = synth.random_problem(seed, 301, kind="matern52", p_missing=0.25, ties=2)
        m = ssm.build(w.components)
        k0, n = sharded.split(w.N, world)[rank]
        be = OracleShard(m, w.noise_var, w.t, w.y, w.mask, k0, n, w.N)
        be.rank = rank
        mean, var, nll = sharded.sharded_posterior(be, sharded.torch_exchange, rank, world)
        q.put((rank, k0, mean.numpy(), var.numpy(), float(nll[0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 17, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    res.sort()
    w = synth.random_problem(17, 301, kind="matern52", p_missing=0.25, ties=2)
    o = oracle.posterior(w)
    mean = np.concatenate([r[2] for r in res]); var = np.concatenate([r[3] for r in res])
    nll = res[0][4]
    assert all(r[4] == nll for r in res)                            # every rank forms the same total
    assert np.max(np.abs(mean - o["mean"])) / np.max(np.abs(o["mean"])) < 1e-9
    assert np.max(np.abs(var - o["var"]) / o["var"]) < 1e-9
    assert abs(nll - o["nll"]) < 1e-9 * abs(o["nll"])


def test_split():
    from paper_2102_09964_b200 import sharded
    for N, W in [(10, 3), (7, 8), (2 ** 20 + 3, 8)]:
        parts = sharded.split(N, W)
        assert sum(n for _, n in parts) == N
        assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(W - 1))
        assert max(n for _, n in parts) - min(n for _, n in parts) <= 1
