"""Small invocations of every hot-path entry point, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): thread path (d = 3, many CTAs, the K3 ticket / flag protocol), NLL-only,
Matern and general-model gradients, the wide path (d = 6 quarter kernels, d = 16, irregular
per-step discretisation), batched series, the fused single pass and virtual sharding.
usage: python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_2102_09964_b200 as P
from paper_2102_09964_b200 import sharded


def dev(w):
    return tuple(torch.from_numpy(a).to("cuda:0") for a in (w.t, w.y, w.mask))


def run(w, chain_len=0, grad=False):
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt, chain_len=chain_len)
    t, y, mk = dev(w)
    mean, var, nll = m.posterior(t, y, mk)
    nll2 = torch.zeros(1, dtype=torch.float64, device="cuda:0")
    P.pssgp_nll(m.h, w.N, t, y, mk, nll2)
    if grad:
        m.nll_grad(t, y, mk)
    m.check()
    torch.cuda.synchronize()
    print(f"{w.name}: N={w.N} d={m.state_dim} nll={float(nll.cpu()[0]):.6f}", flush=True)


run(synth.random_problem(1, 20000, kind="matern52", p_missing=0.2, ties=3), chain_len=5, grad=True)
run(synth.metric_workload(50000))
run(synth.config3(n=3000), chain_len=17, grad=True)
run(synth.config3(n=3000, irregular=True))
run(synth.config4(n=700), grad=True)
run(synth.co2_product(n=600, order=1), grad=True)
w = synth.random_problem(2, 9000, kind="matern32", p_missing=0.3)
mean, var, nll = sharded.run_virtual(w.components, w.noise_var, w.t, w.y, w.mask, 3)
print("virtual sharding G=3 ok", flush=True)
# batched series
m = P.Model(w.components, w.noise_var)
B = 4
off = torch.tensor([0, 1000, 3000, 3001, 9000], dtype=torch.int64, device="cuda:0")
t, y, mk = dev(w)
mean = torch.empty(w.N, dtype=torch.float64, device="cuda:0")
var = torch.empty_like(mean)
nllb = torch.empty(B, dtype=torch.float64, device="cuda:0")
gb = torch.empty(3 * B, dtype=torch.float64, device="cuda:0")
tb = t.clone()
for s, e in ((0, 1000), (1000, 3000), (3000, 3001), (3001, 9000)):
    tb[s:e] -= tb[s].clone()
P.pssgp_posterior_batched(m.h, B, off, None, None, None, w.N, tb, y, mk, mean, var, nllb)
P.pssgp_nll_grad_batched(m.h, B, off, None, None, None, w.N, tb, y, mk, nllb, gb)
m.check()
torch.cuda.synchronize()
print("batched ok", flush=True)
