import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2102_09964_b200 as P
w = synth.random_problem(60, 3200, kind="matern52", p_missing=0.1)
m = P.Model(w.components, w.noise_var)
t, y, mk = (torch.from_numpy(a).cuda() for a in (w.t, w.y, w.mask))
for _ in range(5):
    m.posterior(t, y, mk)
    m.nll_grad(t, y, mk)
torch.cuda.synchronize()
