"""Print GPU-vs-oracle gradient errors (f1) for a few workloads (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2102_09964_b200 as P
from oracle import grad as og

for kind in ["matern12", "matern32", "matern52"]:
    for N in [1000, 20011]:
        w = synth.random_problem(N % 89, N, kind=kind, p_missing=0.3, ties=3)
        c = w.components[0]
        nr, gr = og.kf_nll_grad(kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
        m = P.Model(w.components, w.noise_var)
        t, y, mk = (torch.from_numpy(a).cuda() for a in (w.t, w.y, w.mask))
        nll, g = m.nll_grad(t, y, mk)
        g = g.cpu().numpy()
        print(kind, N, "nll", float(nll.cpu()[0]), nr, "g", g, gr, "rel", np.abs(g - gr) / np.abs(gr))
