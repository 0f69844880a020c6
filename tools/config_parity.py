"""Full-size parity of a BASELINE config on one GPU against the sequential oracle:
python tools/config_parity.py c3            (RBF-6, N = 2^22, uniform dt)
python tools/config_parity.py c3i           (RBF-6, N = 2^22, jittered dt: per-step (F, Q) path)
python tools/config_parity.py c4 [N]        (periodic J=6 + Matern-3/2, d = 16; default N = 2^20)
python tools/config_parity.py c2            (Matern-5/2, 2^20 + 10^4 test points)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import synth
import paper_2102_09964_b200 as P

cfg = sys.argv[1]
if cfg == "c3":
    w = synth.config3()
elif cfg == "c3i":
    w = synth.config3(irregular=True)
elif cfg == "c4":
    w = synth.config4(n=int(sys.argv[2]) if len(sys.argv) > 2 else 2 ** 20)
elif cfg == "c2":
    w = synth.config2()
else:
    raise SystemExit(__doc__)
m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
t, y, mk = (torch.from_numpy(a).cuda() for a in (w.t, w.y, w.mask))
mean, var, nll = m.posterior(t, y, mk)
m.check()
torch.cuda.synchronize()
gm, gv, gn = mean.cpu().numpy(), var.cpu().numpy(), float(nll.cpu()[0])
t0 = time.time()
o = oracle.posterior(w)
em = np.max(np.abs(gm - o["mean"])) / np.max(np.abs(o["mean"]))
ev = np.max(np.abs(gv - o["var"]) / o["var"])
en = abs(gn - o["nll"]) / abs(o["nll"])
ok = em <= 1e-8 and ev <= 1e-8 and en <= 1e-9
print(f"{w.name} N={w.N} d={m.state_dim}: oracle {time.time() - t0:.0f} s; parity mean {em:.3e} var {ev:.3e} "
      f"nll {en:.3e} -> {'PASS' if ok else 'FAIL'}", flush=True)
