"""Small-N latency vs chain length, with the per-kernel split (CUDA events on the launch stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2102_09964_b200 as P


def timeit(fn, reps=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


Ks = [int(a) for a in os.environ.get("KS", "0,1,2,4,8,16,32").split(",")]
Ns = [int(a) for a in os.environ.get("NS", "1200,3200").split(",")]
for n in Ns:
    w = synth.random_problem(60, n, kind="matern52", p_missing=0.1)
    for K in Ks:
        m = P.Model(w.components, w.noise_var, chain_len=K)
        s = torch.cuda.current_stream()
        t, y, mk = (torch.from_numpy(a).cuda() for a in (w.t, w.y, w.mask))
        mean = torch.empty_like(t); var = torch.empty_like(t)
        nll = torch.zeros(1, dtype=torch.float64, device="cuda:0")
        post = lambda: P.pssgp_posterior(m.h, n, t, y, mk, mean, var, nll, s)
        d = timeit(post)
        P.pssgp_profile_enable(m.h, True)
        P.pssgp_profile_read(m.h)
        for _ in range(50):
            post()
        prof = P.pssgp_profile_read(m.h)
        P.pssgp_profile_enable(m.h, False)
        split = {k: round(v[0] / 50 * 1e3, 1) for k, v in prof.items() if v[1] > 0}
        pl = m.plan(n)
        print(f"N={n} K={pl['chain_len']} nb={pl['n_blocks']}: {d:.1f} us/call  split(us) {split}", flush=True)
        m.close()
