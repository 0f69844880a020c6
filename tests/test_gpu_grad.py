"""GPU parity of pssgp_nll_grad (NEXT row f1) against the gradient oracles
(oracle/grad.py): complex-step sequential filter for N up to a few 10^4 and the
dense R&W Eq. (5.9) gradient for small N.

Tolerance: each component g_j is a sum of N per-step terms of either
sign, so a component can be small against the others; the bar is per component,
    |g_gpu,j - g_ref,j| <= GRAD_TOL * (|g_ref,j| + 1e-3 max_i |g_ref,i|) + 1e-12
with GRAD_TOL = 1e-9 (measured errors ~1e-15 relative to |g_ref,j|, tools/grad_errors.py): a
component is checked to 9 digits unless it is below 1e-3 of the largest, and then to 12 digits of
the largest."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import grad as og
import paper_2102_09964_b200 as P

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-9
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
    assert abs(nll - nll_r) <= NLL_TOL * max(abs(nll_r), 1.0), (nll, nll_r)
    err = grad_err(g, g_r)
    assert np.all(err <= GRAD_TOL), (g, g_r, err)
    return err


def grad_err(g, g_r):
    """Per-component error in units of the bar (see the module docstring)."""
    scale = np.abs(g_r) + 1e-3 * np.max(np.abs(g_r)) + 1e-12 / GRAD_TOL
    return np.abs(g - g_r) / scale


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


def _batched_problem(kind, lens, seed=31):
    rng = np.random.default_rng(seed)
    ws = []
    for b, n in enumerate(lens):
        ws.append(synth.random_problem(200 + b, n, kind=kind, p_missing=0.2, ties=min(2, n // 10),
                                       lengthscale=float(rng.uniform(0.2, 2.0)), variance=float(rng.uniform(0.5, 3.0)),
                                       noise_var=float(rng.uniform(0.01, 0.3))) if n > 0 else None)
    return ws


@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
@pytest.mark.parametrize("chain_len", [1, 7, 64, 4096])
def test_grad_batched(cuda_device, kind, chain_len):
    """NEXT rows f1 x f2: per-series NLL and gradient w.r.t. each series' own
    (log sigma_b^2, log ell_b, log sigma_n,b^2), one launch sequence for all series
    (empty, 1-point, in-chain and chain-spanning series), each against the complex-step
    oracle on that series alone."""
    lens = [0, 1, 2, 37, 3200, 0, 5000, 777, 1, 9000, 300]
    ws = _batched_problem(kind, lens)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cat = lambda f, dt: np.concatenate([f(w) if w is not None else np.zeros(0, dt) for w in ws])  # noqa: E731
    t = cat(lambda w: w.t, np.float64); y = cat(lambda w: w.y, np.float64); mk = cat(lambda w: w.mask, np.uint8)
    var_b = np.array([w.components[0].variance if w else 1.0 for w in ws])
    ell_b = np.array([w.components[0].lengthscale if w else 1.0 for w in ws])
    r_b = np.array([w.noise_var if w else 0.1 for w in ws])
    m = P.Model([synth.Component(kind, 1.0, 1.0)], 0.1, chain_len=chain_len)
    dev = "cuda:0"
    T, Y, MK = (torch.from_numpy(a).to(dev) for a in (t, y, mk))
    OFF, VB, EB, RB = (torch.from_numpy(a).to(dev) for a in (off, var_b, ell_b, r_b))
    B = len(lens)
    nll = torch.empty(B, dtype=torch.float64, device=dev)
    g = torch.empty(3 * B, dtype=torch.float64, device=dev)
    P.pssgp_nll_grad_batched(m.h, B, OFF, VB, EB, RB, t.shape[0], T, Y, MK, nll, g)
    m.check()
    nll, g = nll.cpu().numpy(), g.cpu().numpy().reshape(B, 3)
    for b, w in enumerate(ws):
        if w is None:
            assert nll[b] == 0.0 and np.all(g[b] == 0.0)
            continue
        c = w.components[0]
        nll_r, g_r = og.kf_nll_grad(c.kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
        nobs = int(w.mask.sum())
        assert abs(nll[b] - nll_r) <= NLL_TOL * max(abs(nll_r), 1.0), (b, nll[b], nll_r)
        err = np.abs(g[b] - g_r) / (np.abs(g_r) + nobs + 1)
        assert np.all(err <= GRAD_TOL), (b, g[b], g_r, err)


def test_grad_batched_single_series_equals_nll_grad(cuda_device):
    """One series with the model's own hyper-parameters (null per-series arrays) gives
    exactly the single-series entry point's result."""
    w = synth.random_problem(8, 30011, kind="matern52", p_missing=0.15, ties=3)
    m = P.Model(w.components, w.noise_var)
    dev = "cuda:0"
    t, y, mk = (torch.from_numpy(a).to(dev) for a in (w.t, w.y, w.mask))
    nll1, g1 = m.nll_grad(t, y, mk)
    off = torch.tensor([0, w.t.shape[0]], dtype=torch.int64, device=dev)
    nll = torch.empty(1, dtype=torch.float64, device=dev)
    g = torch.empty(3, dtype=torch.float64, device=dev)
    P.pssgp_nll_grad_batched(m.h, 1, off, None, None, None, w.t.shape[0], t, y, mk, nll, g)
    m.check()
    assert abs(float(nll.cpu()[0]) - float(nll1.cpu()[0])) <= 1e-12 * abs(float(nll1.cpu()[0]))
    np.testing.assert_allclose(g.cpu().numpy(), g1.cpu().numpy(), rtol=1e-11, atol=1e-9)


def test_grad_batched_unsupported_model(cuda_device):
    w = synth.config3()
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
    n = 64
    t, y, mk = (torch.from_numpy(a[:n]).to("cuda:0") for a in (w.t, w.y, w.mask))
    off = torch.tensor([0, n], dtype=torch.int64, device="cuda:0")
    out = torch.empty(3, dtype=torch.float64, device="cuda:0")
    with pytest.raises(P.PssgpError):
        P.pssgp_nll_grad_batched(m.h, 1, off, None, None, None, n, t, y, mk, out[:1], out)


def test_grad_batched_invalid_offsets_and_missing_series(cuda_device):
    """Offsets that do not partition [0, N) -> PSSGP_E_INPUT; an all-missing series has NLL 0 and
    gradient 0 while its neighbours stay exact."""
    from paper_2102_09964_b200 import _native
    dev = "cuda:0"
    m = P.Model([synth.Component("matern32", 1.0, 0.5)], 0.01, chain_len=16)
    n = 1000
    t = torch.linspace(0, 1, n, dtype=torch.float64, device=dev)
    y = torch.zeros(n, dtype=torch.float64, device=dev)
    mk = torch.ones(n, dtype=torch.uint8, device=dev)
    nll = torch.empty(2, dtype=torch.float64, device=dev)
    g = torch.empty(6, dtype=torch.float64, device=dev)
    for bad in ([0, 600, 900], [0, 700, 300], [5, 500, n]):
        off = torch.tensor(bad, dtype=torch.int64, device=dev)
        P.pssgp_nll_grad_batched(m.h, 2, off, None, None, None, n, t, y, mk, nll, g)
        with pytest.raises(P.PssgpError) as e:
            m.check()
        assert e.value.status == _native.PSSGP_E_INPUT
    ws = _batched_problem("matern32", [700, 500, 900], seed=5)
    ws[1].mask[:] = 0
    off = np.array([0, 700, 1200, 2100], np.int64)
    T, Y, MK = (torch.from_numpy(np.concatenate([getattr(w, a) for w in ws])).to(dev) for a in ("t", "y", "mask"))
    VB, EB, RB = (torch.tensor([f(w) for w in ws], dtype=torch.float64, device=dev) for f in
                  (lambda w: w.components[0].variance, lambda w: w.components[0].lengthscale, lambda w: w.noise_var))
    nll = torch.empty(3, dtype=torch.float64, device=dev)
    g = torch.empty(9, dtype=torch.float64, device=dev)
    P.pssgp_nll_grad_batched(m.h, 3, torch.from_numpy(off).to(dev), VB, EB, RB, 2100, T, Y, MK, nll, g)
    m.check()
    nll, g = nll.cpu().numpy(), g.cpu().numpy().reshape(3, 3)
    assert nll[1] == 0.0 and np.all(g[1] == 0.0)
    for b in (0, 2):
        w = ws[b]
        c = w.components[0]
        nll_r, g_r = og.kf_nll_grad(c.kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
        assert abs(nll[b] - nll_r) <= NLL_TOL * max(abs(nll_r), 1.0)
        assert np.all(np.abs(g[b] - g_r) / (np.abs(g_r) + w.mask.sum() + 1) <= GRAD_TOL)


# ---------------------------------------------------------------- any model (reverse mode, uniform grids)
GENERAL = {
    # the paper's CO2 model C_Per x C_Mat + C_Mat, n_x = 10 / 14 / 18, weekly grid
    "co2_J1": lambda n: synth.co2_product(n=n, order=1),
    "co2_J2": lambda n: synth.co2_product(n=n, order=2),
    "co2_J3": lambda n: synth.co2_product(n=n, order=3),
    # BASELINE C4 shape: periodic J = 6 + Matern-3/2 trend (d = 16), weekly cadence
    "c4": lambda n: synth.config4(n=n),
    # C3 shape: RBF Taylor order 6 (d = 6), uniform fine grid
    "c3": lambda n: synth.config3(n=n),
    # d <= 3 models other than one Matern component
    "rbf3": lambda n: _uniform_w([synth.Component("rbf", 1.3, 0.8, order=3)], 0.02, n, 0.01),
    "m12+m12": lambda n: _uniform_w([synth.Component("matern12", 1.0, 0.3), synth.Component("matern12", 0.5, 3.0)],
                                    0.05, n, 0.02),
    "per1+m32_sum": lambda n: _uniform_w([synth.Component("periodic", 1.5, 1.0, period=0.7, order=1),
                                          synth.Component("matern32", 1.0, 2.0)], 0.05, n, 0.013),
}


def _uniform_w(comps, r, n, dt, seed=4):
    t = np.arange(n, dtype=np.float64) * dt
    rng = np.random.default_rng(seed)
    mask = (rng.random(n) >= 0.15).astype(np.uint8)
    y = synth.sinusoid(t) + np.sqrt(r) * rng.standard_normal(n)
    y[mask == 0] = np.nan
    return synth.Workload("uniform", comps, r, t, y, mask, uniform_dt=dt)


def assert_grad_general(w, **kw):
    nll_r, g_r = og.kf_nll_grad_general(w.components, w.noise_var, w.t, w.y, w.mask)
    nll, g = gpu_grad(w, **kw)
    assert g.shape == g_r.shape == (len(og.param_names(w.components)),)
    assert abs(nll - nll_r) <= NLL_TOL * max(abs(nll_r), 1.0), (nll, nll_r)
    err = grad_err(g, g_r)
    assert np.all(err <= GRAD_TOL), (g, g_r, err)


@pytest.mark.parametrize("name,n", [("co2_J1", 3192), ("co2_J2", 3192), ("co2_J3", 3192), ("c4", 2000),
                                    ("c3", 3001), ("rbf3", 2500), ("m12+m12", 2500), ("per1+m32_sum", 2500)])
def test_grad_general_models(cuda_device, name, n):
    """f1 widened: the paper's HMC model (CO2 product), the C4 sum,
    RBF, and d <= 3 sums against the complex-step oracle of any SSM."""
    assert_grad_general(GENERAL[name](n))


@pytest.mark.parametrize("chain_len", [1, 7, 64])
def test_grad_general_chain_lengths(cuda_device, chain_len):
    """Many chains: the reverse scan of the chain adjoint maps over several levels."""
    assert_grad_general(GENERAL["co2_J1"](1500), chain_len=chain_len)


def test_grad_general_ties_and_edges(cuda_device):
    """dt = 0 steps (no theta dependence, adjoint passes through), first point missing, N = 1, 2."""
    w = GENERAL["per1+m32_sum"](700)
    w.t[100:104] = w.t[100]
    w.t[104:] -= 3 * w.uniform_dt
    w.mask[0] = 0
    w.y[0] = np.nan
    assert_grad_general(w, chain_len=5)
    for n in (1, 2, 3):
        w = GENERAL["per1+m32_sum"](n)
        w.mask[:] = 1
        w.y = synth.sinusoid(w.t)
        assert_grad_general(w)


def test_grad_general_needs_uniform_grid(cuda_device):
    comps = [synth.Component("rbf", 1.0, 0.5, order=4)]
    w = _uniform_w(comps, 0.02, 100, 0.01)
    m = P.Model(comps, 0.02)                         # no uniform_dt: per-step device discretisation
    t, y, mk = (torch.from_numpy(a).to("cuda:0") for a in (w.t, w.y, w.mask))
    with pytest.raises(P.PssgpError) as e:
        m.nll_grad(t, y, mk)
    assert e.value.status == 6                       # PSSGP_E_UNSUPPORTED


# ---------------------------------------------------------------- batched series, per-series theta
BT_MODELS = {
    "co2_J1": [synth.Component("quasiperiodic", 2.0, 1.0, period=52.0, order=1, mat_lengthscale=300.0, mat_nu2=3),
               synth.Component("matern32", 10.0, 1040.0)],
    "co2_J2": [synth.Component("quasiperiodic", 2.0, 1.0, period=52.0, order=2, mat_lengthscale=300.0, mat_nu2=3),
               synth.Component("matern32", 10.0, 1040.0)],
    "per3+m52": [synth.Component("periodic", 1.5, 0.8, period=40.0, order=3), synth.Component("matern52", 1.0, 60.0)],
    "m12+m32": [synth.Component("matern12", 1.0, 30.0), synth.Component("matern32", 0.5, 200.0)],
    "quasi_m12": [synth.Component("quasiperiodic", 1.0, 0.9, period=30.0, order=2, mat_lengthscale=100.0, mat_nu2=1)],
}


def _batched_theta_problem(name, lens=(1, 2, 300, 701, 1200), seed=3):
    """Series on a weekly grid (dt = 1 week), each with its own log hyper-parameters near the base."""
    comps = BT_MODELS[name]
    rng = np.random.default_rng(seed)
    th0 = og.theta0(comps, 0.09)
    ts, ys, ms, thetas = [], [], [], []
    for i, n in enumerate(lens):
        t = 17.0 * i + np.arange(n, dtype=np.float64)
        mask = (rng.random(n) > 0.1).astype(np.uint8)
        y = synth.co2_like(t / 52.0) + 0.3 * rng.standard_normal(n)
        y[mask == 0] = np.nan
        ts.append(t); ys.append(y); ms.append(mask)
        thetas.append(th0 + rng.uniform(-0.25, 0.25, th0.shape[0]))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return comps, ts, ys, ms, np.array(thetas), off


@pytest.mark.parametrize("name", list(BT_MODELS))
def test_batched_theta_grad_and_posterior(cuda_device, name):
    """Per-series hyper-parameters for sums of Matern / periodic / quasi-periodic components (the
    paper's HMC chains on the CO2 model): each series against the oracle at its own theta
    (complex-step gradient; sequential KF + RTS posterior)."""
    comps, ts, ys, ms, thetas, off = _batched_theta_problem(name)
    B, npar = thetas.shape
    m = P.Model(comps, 0.09, uniform_dt=1.0)
    assert m.num_params == npar
    dev = "cuda:0"
    t = torch.from_numpy(np.concatenate(ts)).to(dev)
    y = torch.from_numpy(np.concatenate(ys)).to(dev)
    mk = torch.from_numpy(np.concatenate(ms)).to(dev)
    N = int(t.shape[0])
    offd = torch.from_numpy(off).to(dev)
    th = torch.from_numpy(np.ascontiguousarray(thetas)).to(dev)
    nll = torch.zeros(B, dtype=torch.float64, device=dev)
    grad = torch.zeros(B * npar, dtype=torch.float64, device=dev)
    P.pssgp_nll_grad_batched_theta(m.h, B, offd, th, N, t, y, mk, nll, grad)
    mean = torch.zeros(N, dtype=torch.float64, device=dev)
    var = torch.zeros(N, dtype=torch.float64, device=dev)
    nll2 = torch.zeros(B, dtype=torch.float64, device=dev)
    P.pssgp_posterior_batched_theta(m.h, B, offd, th, N, t, y, mk, mean, var, nll2)
    m.check()
    g = grad.cpu().numpy().reshape(B, npar)
    nl, nl2, mean, var = nll.cpu().numpy(), nll2.cpu().numpy(), mean.cpu().numpy(), var.cpu().numpy()
    for b in range(B):
        cb, rb = og.components_at(comps, thetas[b])
        nll_r, g_r = og.kf_nll_grad_general(cb, rb, ts[b], ys[b], ms[b])
        assert abs(nl[b] - nll_r) <= NLL_TOL * max(abs(nll_r), 1.0), (b, nl[b], nll_r)
        assert nl2[b] == nl[b]
        err = grad_err(g[b], g_r)
        assert np.all(err <= GRAD_TOL), (b, g[b], g_r, err)
        o = oracle.posterior(synth.Workload("bt", cb, rb, ts[b], ys[b], ms[b]))
        sl = slice(off[b], off[b + 1])
        assert np.max(np.abs(mean[sl] - o["mean"])) <= 1e-8 * max(np.max(np.abs(o["mean"])), 1e-300)
        assert np.max(np.abs(var[sl] - o["var"]) / o["var"]) <= 1e-8


def test_batched_theta_rejects_rbf_and_irregular(cuda_device):
    comps = [synth.Component("rbf", 1.0, 0.5, order=4)]
    m = P.Model(comps, 0.02, uniform_dt=0.01)
    dev = "cuda:0"
    t = torch.arange(10, dtype=torch.float64, device=dev) * 0.01
    y = torch.zeros(10, dtype=torch.float64, device=dev)
    mk = torch.ones(10, dtype=torch.uint8, device=dev)
    off = torch.tensor([0, 10], dtype=torch.int64, device=dev)
    th = torch.zeros((1, m.num_params), dtype=torch.float64, device=dev)
    nll = torch.zeros(1, dtype=torch.float64, device=dev)
    with pytest.raises(P.PssgpError) as e:
        P.pssgp_posterior_batched_theta(m.h, 1, off, th, 10, t, y, mk, None, None, nll)
    assert e.value.status == 6
    # a non-uniform step inside a series is reported by pssgp_check
    m = P.Model([synth.Component("matern32", 1.0, 0.5), synth.Component("matern12", 1.0, 2.0)], 0.02, uniform_dt=0.01)
    th = torch.from_numpy(og.theta0(m_comps := [synth.Component("matern32", 1.0, 0.5),
                                                synth.Component("matern12", 1.0, 2.0)], 0.02)[None, :]).to(dev)
    t2 = t.clone()
    t2[5:] += 0.003
    P.pssgp_posterior_batched_theta(m.h, 1, off, th, 10, t2, y, mk, None, None, nll)
    with pytest.raises(P.PssgpError) as e:
        m.check()
    assert e.value.status == 6
