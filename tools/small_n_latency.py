"""Latency of one call at the paper's dataset sizes (N = 1,200 C1 and 3,200 sunspots): direct
launches vs a CUDA-graph replay of the same call (the K3 carry flag makes replays safe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2102_09964_b200 as P


def timeit(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


for n in (1200, 3200):
    w = synth.random_problem(60, n, kind="matern52", p_missing=0.1)
    m = P.Model(w.components, w.noise_var)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        t, y, mk = (torch.from_numpy(a).cuda() for a in (w.t, w.y, w.mask))
        mean = torch.empty_like(t); var = torch.empty_like(t)
        nll = torch.zeros(1, dtype=torch.float64, device="cuda:0")
        grad = torch.zeros(3, dtype=torch.float64, device="cuda:0")
        post = lambda: P.pssgp_posterior(m.h, n, t, y, mk, mean, var, nll, s)
        ngr = lambda: P.pssgp_nll_grad(m.h, n, t, y, mk, nll, grad, s)
        d_post, d_grad = timeit(post), timeit(ngr)
        gp, gg = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gp, stream=s):
            post()
        with torch.cuda.graph(gg, stream=s):
            ngr()
        g_post, g_grad = timeit(gp.replay), timeit(gg.replay)
    print(f"N={n}: posterior {d_post:.1f} us direct, {g_post:.1f} us graph; NLL+grad {d_grad:.1f} us direct, "
          f"{g_grad:.1f} us graph", flush=True)
