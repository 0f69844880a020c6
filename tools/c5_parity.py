"""Full-size C5 shape (N = 2^27, Matern-5/2, jittered, 1/16 missing) on ONE GPU:
time the posterior and compare every output with the sequential oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2102_09964_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 27
w = synth.metric_workload(n)
m = P.Model(w.components, w.noise_var)
t, y, mk = (torch.from_numpy(a).cuda() for a in (w.t, w.y, w.mask))
mean, var, nll = m.posterior(t, y, mk)
m.check(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    m.posterior(t, y, mk, out=(mean, var, nll))
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"N={n} gpu {ms:.2f} ms/step = {n / ms / 1e6:.2f} G steps/s", flush=True)
gm, gv, gn = mean.cpu().numpy(), var.cpu().numpy(), float(nll.cpu()[0])
del t, y, mk, mean, var
t0 = time.time()
o = oracle.posterior(w)
print(f"oracle {time.time() - t0:.0f} s", flush=True)
em = np.max(np.abs(gm - o["mean"])) / np.max(np.abs(o["mean"]))
ev = np.max(np.abs(gv - o["var"]) / o["var"])
en = abs(gn - o["nll"]) / abs(o["nll"])
print(f"parity: mean {em:.3e} var {ev:.3e} nll {en:.3e}  ->", "PASS" if em <= 1e-8 and ev <= 1e-8 and en <= 1e-9 else "FAIL")
