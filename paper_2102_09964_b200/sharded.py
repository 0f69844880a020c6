"""Time-sharded multi-GPU driver.

One process per GPU; rank g owns the contiguous chunk [k0_g, k0_g + n_g) of
the global grid.  The exchange is the paper's associativity (PAPER.md:326,
431: any grouping of the scan is allowed) applied across devices:

  1. filter reduce : each rank folds its chunk into ONE filter aggregate
                     (A, b, C, eta, J)                       -> all_gather
  2. filter apply  : rank g applies the ordered product of aggregates 0..g-1
                     (a collapsed global prefix, A = 0 after rank 0's element
                     with A_1 = 0, Eq. (7)), runs the Kalman rescan, emits ONE
                     smoother blob = its smoother aggregate (E, g, L) followed by
                     its NLL partial                        -> all_gather
  3. smoother apply: rank g applies the ordered product of smoother aggregates
                     g+1..G-1 (collapsed global suffix), runs the RTS rescan; the
                     library forms the total NLL as the fixed-order sum of the
                     gathered partials (deterministic, identical on every rank).
  Two collectives per posterior; the binding does no arithmetic.

The collectives carry a few hundred bytes (27 + 18 + 1 doubles at d = 3), so
they are latency-bound; NCCL over NVLink/NVSwitch through torch.distributed.
Arithmetic happens only inside libpssgp.so kernels.  The protocol itself
(`sharded_posterior`) is backend-agnostic so the CPU test suite can drive it
with gloo and a mock backend.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np

from . import (Model, pssgp_aggregate_bytes, pssgp_shard_filter_apply, pssgp_shard_filter_reduce,
               pssgp_shard_smoother_apply)


def split(N: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous chunks (k0, n) of near-equal size (all steps cost the same)."""
    base, rem = divmod(N, world)
    out, k0 = [], 0
    for g in range(world):
        n = base + (1 if g < rem else 0)
        out.append((k0, n))
        k0 += n
    return out


def sharded_posterior(backend, exchange: Callable, rank: int, world: int):
    """Backend-agnostic 3-phase protocol.

    backend.filter_reduce() -> filter aggregate blob
    backend.filter_apply(all_filter_blobs) -> smoother blob (aggregate + NLL partial)
    backend.smoother_apply(all_smoother_blobs) -> (mean, var, total NLL)
    exchange(x) -> stacked [world, ...] in rank order
    """
    fa = backend.filter_reduce()
    all_fa = exchange(fa)
    sb = backend.filter_apply(all_fa)
    all_sb = exchange(sb)
    return backend.smoother_apply(all_sb)


class DeviceShard:
    """libpssgp.so backend for one rank: t_full must hold the chunk plus its halo."""

    def __init__(self, model: Model, t, y, mask, k0: int, n: int, N: int, rank: int, world: int, stream=None):
        import torch
        self.m, self.k0, self.n, self.N, self.rank, self.world = model, k0, n, N, rank, world
        self.t, self.y, self.mask = t, y, mask      # device tensors: t[k0-1 .. k0+n] accessible via offset
        self.t_off = 1 if k0 > 0 else 0             # index of local step 0 inside self.t
        self.stream = stream
        dev = t.device
        self.fbytes = pssgp_aggregate_bytes(model.h, 0)
        self.sbytes = pssgp_aggregate_bytes(model.h, 1)
        self.fagg = torch.zeros(self.fbytes // 8, dtype=torch.float64, device=dev)
        self.sagg = torch.zeros(self.sbytes // 8, dtype=torch.float64, device=dev)   # aggregate + NLL partial
        self.nll = torch.zeros(1, dtype=torch.float64, device=dev)                    # total NLL (all ranks)
        self.mean = torch.empty(n, dtype=torch.float64, device=dev)
        self.var = torch.empty(n, dtype=torch.float64, device=dev)

    def _tp(self):
        return int(self.t.data_ptr()) + 8 * self.t_off

    def filter_reduce(self):
        pssgp_shard_filter_reduce(self.m.h, self.k0, self.n, self.N, self._tp(), int(self.y.data_ptr()),
                                  int(self.mask.data_ptr()), int(self.fagg.data_ptr()), self.stream)
        return self.fagg

    def filter_apply(self, all_fa):
        pssgp_shard_filter_apply(self.m.h, self.k0, self.n, self.N, self._tp(), int(self.y.data_ptr()),
                                 int(self.mask.data_ptr()), int(all_fa.data_ptr()), self.rank, self.world,
                                 int(self.sagg.data_ptr()), None, self.stream)
        return self.sagg

    def smoother_apply(self, all_sb):
        pssgp_shard_smoother_apply(self.m.h, self.k0, self.n, self.N, self._tp(), int(all_sb.data_ptr()),
                                   self.rank, self.world, int(self.mean.data_ptr()), int(self.var.data_ptr()),
                                   int(self.nll.data_ptr()), self.stream)
        return self.mean, self.var, self.nll


def torch_exchange(x):
    """all_gather of a 1-D tensor into [world, len] in rank order (NCCL: one
    all_gather_into_tensor over NVLink; gloo: list all_gather, for CPU tests)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    x = x.contiguous()
    if dist.get_backend() == "nccl":
        out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x)
        return out
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x)
    return torch.stack(parts)


nccl_exchange = torch_exchange


def chunk_inputs(t: np.ndarray, y: np.ndarray, mask: np.ndarray, k0: int, n: int, device):
    """Host -> device copy of one rank's chunk with its one-point halo of t."""
    import torch
    lo = max(k0 - 1, 0)
    hi = min(k0 + n + 1, t.shape[0])
    tt = torch.from_numpy(np.ascontiguousarray(t[lo:hi])).to(device)
    yy = torch.from_numpy(np.ascontiguousarray(y[k0:k0 + n])).to(device)
    mm = torch.from_numpy(np.ascontiguousarray(mask[k0:k0 + n])).to(device)
    return tt, yy, mm


def run_virtual(components: Sequence, noise_var: float, t: np.ndarray, y: np.ndarray, mask: np.ndarray,
                world: int, uniform_dt: float = 0.0, device: str = "cuda:0"):
    """All ranks' shard phases run one after another on ONE GPU (no kernel waits
    on another); the 'exchange' is a stack in device memory.  For tests."""
    import torch
    N = t.shape[0]
    parts = split(N, world)
    shards = []
    for g, (k0, n) in enumerate(parts):
        m = Model(components, noise_var, uniform_dt=uniform_dt)
        tt, yy, mm = chunk_inputs(t, y, mask, k0, n, device)
        shards.append(DeviceShard(m, tt, yy, mm, k0, n, N, g, world))
    fa = torch.stack([s.filter_reduce().clone() for s in shards])
    sb = torch.stack([s.filter_apply(fa).clone() for s in shards])
    res = [s.smoother_apply(sb) for s in shards]
    for s in shards:
        s.m.check()
    mean = torch.cat([r[0] for r in res]).cpu().numpy()
    var = torch.cat([r[1] for r in res]).cpu().numpy()
    nlls = [float(r[2].cpu()[0]) for r in res]
    assert all(v == nlls[0] for v in nlls), "total NLL differs between ranks"
    return mean, var, nlls[0]
