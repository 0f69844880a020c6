"""Full-size GPU parity of the BASELINE configurations that only builder logs covered in round 1
("Next round" item 1): every output of the CUDA path (through the C ABI, in the launch
configuration bench.py times) against the sequential fp64 oracle, element by element.

    C3  RBF Taylor order 6 (d = 6), N = 2^22, uniform dt          (BASELINE configs[2])
    C4  periodic J = 6 + Matern-3/2 trend (d = 16), N = 2^24      (BASELINE configs[3])
    C5  Matern-5/2, N = 2^27, jittered times                      (BASELINE configs[4], one GPU)

Tolerances: north_star (mean normwise 1e-8, var elementwise 1e-8, NLL 1e-9; measures of SURVEY.md
§8(c) reading Z14).  The three sequential oracles (5 s, ~230 s and ~285 s on one host core) start
together in a thread pool the first time any of these tests runs (the ctypes calls release the
GIL), so the module costs about as long as the slowest of them.  The measured errors are reported
as ParityReport warnings (visible in the -q summary).
"""
import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2102_09964_b200 as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

MEAN_TOL, VAR_TOL, NLL_TOL = 1e-8, 1e-8, 1e-9


class ParityReport(UserWarning):
    pass


def _workloads():
    return {"C3": lambda: synth.config3(n=2 ** 22),
            "C4": lambda: synth.config4(n=2 ** 24),
            "C5": lambda: synth.metric_workload(2 ** 27)}


@pytest.fixture(scope="module")
def oracle_jobs(request):
    """Workloads and their oracle results (futures) of the SELECTED tests of this module, all
    started at once."""
    names = {"test_config3_full_size": "C3", "test_config4_full_size": "C4", "test_config5_full_size": "C5"}
    selected = {names[it.name] for it in request.session.items if it.name in names}
    ws = {k: f() for k, f in _workloads().items() if k in selected}
    ex = ThreadPoolExecutor(max_workers=max(1, len(ws)))
    futs = {k: ex.submit(oracle.posterior, w) for k, w in ws.items()}
    yield ws, futs
    ex.shutdown(wait=True)


def _check(name, w, fut):
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
    t, y, mk = (torch.from_numpy(a).to("cuda:0") for a in (w.t, w.y, w.mask))
    mean, var, nll = m.posterior(t, y, mk)
    m.check()
    plan = m.plan(w.N)
    gm, gv, gn = mean.cpu().numpy(), var.cpu().numpy(), float(nll.cpu()[0])
    del t, y, mk, mean, var
    o = fut.result()
    em = np.max(np.abs(gm - o["mean"])) / np.max(np.abs(o["mean"]))
    ev = np.max(np.abs(gv - o["var"]) / o["var"])
    en = abs(gn - o["nll"]) / abs(o["nll"])
    warnings.warn(ParityReport(f"{name} N={w.N} d={m.state_dim} chain_len={plan['chain_len']} "
                               f"chains={plan['n_chains']}: mean {em:.2e} var {ev:.2e} nll {en:.2e}"))
    assert em <= MEAN_TOL and ev <= VAR_TOL and en <= NLL_TOL, (name, em, ev, en)


def test_config3_full_size(cuda_device, oracle_jobs):
    ws, futs = oracle_jobs
    _check("C3", ws["C3"], futs["C3"])


def test_config4_full_size(cuda_device, oracle_jobs):
    ws, futs = oracle_jobs
    _check("C4", ws["C4"], futs["C4"])


def test_config5_full_size(cuda_device, oracle_jobs):
    ws, futs = oracle_jobs
    _check("C5", ws["C5"], futs["C5"])
