"""Per-rank device time of the time-sharded protocol's three phases for one rank's chunk of the
metric grid (N = 2^24 split over G ranks), measured on ONE GPU with CUDA events (no collective:
the aggregates of the other ranks are synthetic placeholders of the right shape; only the time is
of interest).  An estimate of the strong-scaling ceiling before collective latency."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2102_09964_b200 as P
from paper_2102_09964_b200 import sharded

N = 2 ** 24
w = synth.metric_workload(N)
for G in (1, 2, 4, 8):
    rank = G - 1 if G > 1 else 0                      # the last rank: all three phases do full work
    k0, n = sharded.split(N, G)[rank]
    m = P.Model(w.components, w.noise_var)
    tt, yy, mm = sharded.chunk_inputs(w.t, w.y, w.mask, k0, n, "cuda:0")
    sh = sharded.DeviceShard(m, tt, yy, mm, k0, n, N, rank, G)
    fa = sh.filter_reduce()
    all_fa = torch.stack([fa.clone() for _ in range(G)])
    all_fa[:rank] = 0.0
    all_fa[:rank, 0::4] = 0.0
    sa = sh.filter_apply(all_fa)
    all_sa = torch.stack([sa.clone() for _ in range(G)])
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    reps = 20
    tot = [0.0, 0.0, 0.0]
    for _ in range(reps):
        e[0].record(); sh.filter_reduce(); e[1].record(); sh.filter_apply(all_fa); e[2].record()
        sh.smoother_apply(all_sa); e[3].record()
        torch.cuda.synchronize()
        for i in range(3):
            tot[i] += e[i].elapsed_time(e[i + 1])
    ms = [x / reps for x in tot]
    print(f"G={G} chunk={n} reduce {ms[0]:.3f} apply {ms[1]:.3f} smooth {ms[2]:.3f} total {sum(ms):.3f} ms", flush=True)

# per-kernel split at G = 8 (profile slots)
P.pssgp_profile_enable(m.h, True)
P.pssgp_profile_read(m.h)
for _ in range(reps):
    sh.filter_reduce(); sh.filter_apply(all_fa); sh.smoother_apply(all_sa)
torch.cuda.synchronize()
prof = P.pssgp_profile_read(m.h)
print({k: round(v[0] / reps, 4) for k, v in prof.items() if v[1]}, "plan", m.plan(n))
