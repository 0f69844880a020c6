"""GPU parity of the optional fp32 path (pssgp_posterior_f32) against the
fp64 CPU oracle.  Bar (north_star "an optional fp32 path must match to 1e-3", measures of
SURVEY.md §8(c) / DESIGN.md reading Z14): mean normwise, var elementwise, NLL relative —
normalised by N_obs when |NLL| < 0.01 N_obs (per-step NLL terms are O(1), reading Z25)."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2102_09964_b200 as P
from paper_2102_09964_b200 import _native

pytestmark = pytest.mark.gpu

F32_TOL = 1e-3


def run_f32(w, **kw):
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt, **kw)
    t, y, mk = (torch.from_numpy(a).to("cuda:0") for a in (w.t, w.y, w.mask))
    mean, var, nll = m.posterior_f32(t, y, mk)
    m.check()
    return mean.cpu().numpy(), var.cpu().numpy(), float(nll.cpu()[0]), m


def f32_errors(w, g, o):
    mean, var, nll = g
    em = np.max(np.abs(mean - o["mean"])) / max(np.max(np.abs(o["mean"])), 1e-300)
    ev = np.max(np.abs(var - o["var"]) / np.abs(o["var"]))
    nobs = int(w.mask.sum())
    scale = abs(o["nll"]) if abs(o["nll"]) >= 0.01 * nobs else max(nobs, 1)
    en = abs(nll - o["nll"]) / scale
    return em, ev, en


def assert_f32(w, **kw):
    o = oracle.posterior(w)
    mean, var, nll, m = run_f32(w, **kw)
    if w.mask.sum() == 0:
        assert np.max(np.abs(mean)) == 0.0 and nll == 0.0
        np.testing.assert_allclose(var, o["var"], rtol=F32_TOL)
        return (0.0, 0.0, 0.0)
    e = f32_errors(w, (mean, var, nll), o)
    assert max(e) <= F32_TOL, e
    return e


@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
@pytest.mark.parametrize("N", [1, 2, 33, 1000, 4099, 30011])
def test_f32_random_sizes(cuda_device, kind, N):
    w = synth.random_problem(N % 97, N, kind=kind, p_missing=0.3, ties=min(3, N // 10))
    assert_f32(w)


def test_f32_config1(cuda_device):
    assert_f32(synth.config1())


def test_f32_config2(cuda_device):
    assert_f32(synth.config2())


@pytest.mark.parametrize("uniform", [False, True])
def test_f32_metric_grid(cuda_device, uniform):
    """The metric's grid density (dt = 1.2e-4, lambda dt = 5.5e-4) at 2^18 steps."""
    assert_f32(synth.metric_workload(2 ** 18, uniform=uniform))


@pytest.mark.parametrize("chain_len", [1, 5, 17])
def test_f32_small_chains(cuda_device, chain_len):
    w = synth.random_problem(5, 70001, kind="matern52", p_missing=0.2, ties=4, dt_scale=0.01)
    assert_f32(w, chain_len=chain_len)


@pytest.mark.parametrize("p_missing,first_missing", [(1.0, None), (0.5, True), (0.97, True)])
def test_f32_missing_patterns(cuda_device, p_missing, first_missing):
    assert_f32(synth.random_problem(8, 3001, kind="matern32", p_missing=p_missing, first_missing=first_missing))


def test_f32_large_gaps(cuda_device):
    assert_f32(synth.random_problem(12, 5000, kind="matern52", p_missing=0.6, dt_scale=0.8, lengthscale=0.3))


@pytest.mark.slow
def test_f32_metric_full_size(cuda_device):
    """Headline configuration N = 2^24 (the f32 bench line's launch configuration)."""
    e = assert_f32(synth.metric_workload(2 ** 24))
    print("f32 full-size errors (mean, var, nll):", e)


def test_f32_nll_only_and_determinism(cuda_device):
    w = synth.random_problem(2, 20000, kind="matern52", p_missing=0.1)
    m = P.Model(w.components, w.noise_var)
    t, y, mk = (torch.from_numpy(a).to("cuda:0") for a in (w.t, w.y, w.mask))
    a = [x.clone() for x in m.posterior_f32(t, y, mk)]
    b = m.posterior_f32(t, y, mk)
    for u, v in zip(a, b):
        assert torch.equal(u, v)
    nll = torch.zeros(1, dtype=torch.float64, device="cuda:0")
    P.pssgp_posterior_f32(m.h, w.N, t, y, mk, None, None, nll)
    m.check()
    assert float(nll.cpu()[0]) == float(a[2].cpu()[0])
    # the fp64 path on the same handle is unaffected (shared workspace)
    mean64, var64, nll64 = m.posterior(t, y, mk)
    o = oracle.posterior(w)
    assert abs(float(nll64.cpu()[0]) - o["nll"]) <= 1e-9 * abs(o["nll"])


def test_f32_input_errors_and_unsupported(cuda_device):
    w = synth.random_problem(6, 5000, kind="matern52", p_missing=0.2)
    t = w.t.copy(); t[3001] = t[3000] - 1e-6
    m = P.Model(w.components, w.noise_var)
    tt = torch.from_numpy(t).cuda()
    _, y, mk = (torch.from_numpy(a).to("cuda:0") for a in (w.t, w.y, w.mask))
    m.posterior_f32(tt, y, mk)
    with pytest.raises(P.PssgpError) as e:
        m.check()
    assert e.value.status == _native.PSSGP_E_INPUT and e.value.index == 3001
    w3 = synth.config3()
    m3 = P.Model(w3.components, w3.noise_var, uniform_dt=w3.uniform_dt)
    t3, y3, k3 = (torch.from_numpy(a[:64]).to("cuda:0") for a in (w3.t, w3.y, w3.mask))
    with pytest.raises(P.PssgpError) as e:
        m3.posterior_f32(t3, y3, k3)
    assert e.value.status == _native.PSSGP_E_UNSUPPORTED


def test_f32_empty_and_plan(cuda_device):
    w = synth.random_problem(3, 100, kind="matern32")
    m = P.Model(w.components, w.noise_var)
    e = torch.empty(0, dtype=torch.float64, device="cuda:0")
    mean, var, nll = m.posterior_f32(e, e, torch.empty(0, dtype=torch.uint8, device="cuda:0"))
    m.check()
    assert float(nll.cpu()[0]) == 0.0
    pl = m.plan(2 ** 24, f32=True)
    assert pl["chain_len"] * pl["n_chains"] >= 2 ** 24 and pl["threads"] == 128
