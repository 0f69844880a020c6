"""GPU parity of pssgp_nll_grad (NEXT row f1) against the gradient oracles
(oracle/grad.py): complex-step sequential filter for N up to a few 10^4 and the
dense R&W Eq. (5.9) gradient for small N.

Tolerance: each component g_j is a sum of N
per-step terms of either sign; fp64 rounding of the tangent recursion gives an
error ~ eps * cond * sum_k |term_k|, so the bar is
    |g_gpu - g_ref| <= GRAD_TOL * (|g_ref| + N_obs)
with GRAD_TOL = 1e-10 (per-step terms are O(1) for these workloads; measured
errors are ~1e-15 relative to |g_ref|, tools/grad_errors.py)."""
import numpy as np
import pytest
import torch

import synth
from oracle import grad as og
import paper_2102_09964_b200 as P

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-10
NLL_TOL = 1e-9


def gpu_grad(w, **kw):
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt, **kw)
    dev = "cuda:0"
    t, y, mk = (torch.from_numpy(a).to(dev) for a in (w.t, w.y, w.mask))
    nll, g = m.nll_grad(t, y, mk)
    m.check()
    return float(nll.cpu()[0]), g.cpu().numpy()


def assert_grad(w, ref=None, **kw):
    c = w.components[0]
    if ref is None:
        ref = og.kf_nll_grad(c.kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
    nll_r, g_r = ref
    nll, g = gpu_grad(w, **kw)
    nobs = int(w.mask.sum())
    assert abs(nll - nll_r) <= NLL_TOL * max(abs(nll_r), 1.0), (nll, nll_r)
    err = np.abs(g - g_r) / (np.abs(g_r) + nobs + 1)
    assert np.all(err <= GRAD_TOL), (g, g_r, err)
    return err


@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
@pytest.mark.parametrize("N", [1, 2, 33, 1000, 20011])
def test_grad_random(cuda_device, kind, N):
    w = synth.random_problem(N % 89, N, kind=kind, p_missing=0.3, ties=min(3, N // 10))
    assert_grad(w)


@pytest.mark.parametrize("chain_len", [1, 3, 16])
def test_grad_small_chains(cuda_device, chain_len):
    """Tiny chains -> many CTAs and a multi-level ordered block reduction."""
    w = synth.random_problem(3, 15001, kind="matern52", p_missing=0.2, ties=4, dt_scale=0.01)
    assert_grad(w, chain_len=chain_len)


@pytest.mark.parametrize("first_missing,p_missing", [(True, 0.5), (False, 0.0), (True, 0.95)])
def test_grad_missing_patterns(cuda_device, first_missing, p_missing):
    w = synth.random_problem(4, 3001, kind="matern32", p_missing=p_missing, first_missing=first_missing)
    assert_grad(w)


def test_grad_dense_reference(cuda_device):
    """Against the textbook dense gradient (Lemma 1), config-1 sized problem."""
    w = synth.config1()
    c = w.components[0]
    ref = og.dense_nll_grad(c.kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
    assert_grad(w, ref=ref)


def test_grad_all_missing_and_empty(cuda_device):
    w = synth.random_problem(6, 500, kind="matern52", p_missing=1.0)
    nll, g = gpu_grad(w)
    assert nll == 0.0 and np.all(g == 0.0)
    m = P.Model(w.components, w.noise_var)
    e = torch.empty(0, dtype=torch.float64, device="cuda:0")
    nll, g = m.nll_grad(e, e, torch.empty(0, dtype=torch.uint8, device="cuda:0"))
    assert float(nll.cpu()[0]) == 0.0 and np.all(g.cpu().numpy() == 0.0)


def test_grad_nll_equals_posterior_nll(cuda_device):
    w = synth.random_problem(7, 50000, kind="matern52", p_missing=0.1)
    nll, _ = gpu_grad(w)
    m = P.Model(w.components, w.noise_var)
    t, y, mk = (torch.from_numpy(a).to("cuda:0") for a in (w.t, w.y, w.mask))
    _, _, nll2 = m.posterior(t, y, mk)
    assert nll == float(nll2.cpu()[0])


def test_grad_unsupported_model(cuda_device):
    w = synth.config3()
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
    t, y, mk = (torch.from_numpy(a[:64]).to("cuda:0") for a in (w.t, w.y, w.mask))
    with pytest.raises(P.PssgpError):
        m.nll_grad(t, y, mk)
