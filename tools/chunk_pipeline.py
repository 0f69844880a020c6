"""Prototype: overlap K1 (fp64-bound fold) of chunk c+1 with K3 (HBM-bound rescan) of chunk c on one
GPU, through the time-sharded phase API (G chunks = G 'virtual ranks', two streams).  Measures
whether the ALU-bound and memory-bound passes co-run profitably before any native pipelining."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_2102_09964_b200 as P
from paper_2102_09964_b200 import sharded

N = int(os.environ.get("N", 2 ** 24))
w = synth.metric_workload(N)
dev = "cuda:0"


def bench(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    for _ in range(reps):
        fn()
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


m0 = P.Model(w.components, w.noise_var)
t, y, mk = (torch.from_numpy(a).to(dev) for a in (w.t, w.y, w.mask))
mean = torch.empty(N, dtype=torch.float64, device=dev); var = torch.empty_like(mean)
nll = torch.zeros(1, dtype=torch.float64, device=dev)
base = bench(lambda: P.pssgp_posterior(m0.h, N, t, y, mk, mean, var, nll, torch.cuda.current_stream()))
print(f"baseline pssgp_posterior: {base:.4f} ms", flush=True)
ref_mean = mean.clone()

for G in (2, 4, 8):
    parts = sharded.split(N, G)
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    shards = []
    for g, (k0, n) in enumerate(parts):
        m = P.Model(w.components, w.noise_var)
        lo = max(k0 - 1, 0)
        tt = t[lo:min(k0 + n + 1, N)]
        shards.append(sharded.DeviceShard(m, tt, y[k0:k0 + n], mk[k0:k0 + n], k0, n, N, g, G))
    fa = torch.zeros((G, shards[0].fbytes // 8), dtype=torch.float64, device=dev)
    sa = torch.zeros((G, shards[0].sbytes // 8), dtype=torch.float64, device=dev)
    evA = [torch.cuda.Event() for _ in range(G)]
    evB = torch.cuda.Event()

    def run(overlap=True):
        cur = torch.cuda.current_stream()
        sA.wait_stream(cur); sB.wait_stream(cur)
        for g, s in enumerate(shards):
            s.stream = sA
            s.filter_reduce()
            fa[g].copy_(s.fagg, non_blocking=True) if False else None
            with torch.cuda.stream(sA):
                fa[g].copy_(s.fagg)
            evA[g].record(sA)
            if not overlap:
                sB.wait_event(evA[g])
        for g, s in enumerate(shards):
            sB.wait_event(evA[g])
            s.stream = sB
            s.filter_apply(fa)
            with torch.cuda.stream(sB):
                sa[g].copy_(s.sagg)
        for s in shards:
            s.stream = sB
            s.smoother_apply(sa)
        cur.wait_stream(sB)

    tp = bench(run)
    err = float((torch.cat([s.mean for s in shards]) - ref_mean).abs().max())
    print(f"G={G}: pipelined {tp:.4f} ms  (max |mean diff| {err:.2e})", flush=True)
