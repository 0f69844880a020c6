"""Pins for the NLL-gradient oracle (oracle/grad.py; NEXT row f1, PAPER.md:77,
157, 173).  Each oracle is checked against something other than itself:
closed forms, finite differences of independently written functions, the
C sequential oracle's NLL, and the other gradient definition (Lemma 1)."""
import math

import numpy as np
import pytest

import oracle
import synth
from oracle import grad as og
from oracle import ssm as ossm
from oracle.dense_gp import dense_gp

KINDS = ["matern12", "matern32", "matern52"]


def richardson(f, x, h):
    """4th-order central difference f'(x)."""
    return (8.0 * (f(x + h) - f(x - h)) - (f(x + 2 * h) - f(x - 2 * h))) / (12.0 * h)


@pytest.mark.parametrize("kind", KINDS)
def test_kernel_dlogell_vs_fd(kind):
    """d k / d log ell against finite differences of oracle.ssm.kernel_value."""
    tau = np.linspace(0.0, 3.0, 31)
    s2, ell = 1.7, 0.6
    nu2 = og._NU2[kind]
    k, dk = og.matern_k_and_dlogell(nu2, s2, ell, tau)
    np.testing.assert_allclose(k, ossm.kernel_value(synth.Component(kind, s2, ell), tau), rtol=1e-14, atol=1e-15)
    fd = richardson(lambda le: ossm.kernel_value(synth.Component(kind, s2, math.exp(le)), tau), math.log(ell), 1e-3)
    np.testing.assert_allclose(dk, fd, rtol=1e-8, atol=1e-11)


def test_single_observation_closed_form():
    """N = 1: NLL = 0.5 log(2 pi S) + y^2 / (2 S), S = s2 + r; gradient by hand."""
    s2, ell, r, y0 = 1.3, 0.7, 0.2, 0.9
    S = s2 + r
    want = np.array([0.5 * s2 / S - 0.5 * y0 * y0 * s2 / S ** 2, 0.0, 0.5 * r / S - 0.5 * y0 * y0 * r / S ** 2])
    t, y, mask = np.array([0.3]), np.array([y0]), np.array([1], np.uint8)
    for kind in KINDS:
        nll_d, g_d = og.dense_nll_grad(kind, s2, ell, r, t, y, mask)
        nll_k, g_k = og.kf_nll_grad(kind, s2, ell, r, t, y, mask)
        assert abs(nll_d - (0.5 * math.log(2 * math.pi * S) + 0.5 * y0 * y0 / S)) < 1e-14
        assert abs(nll_k - nll_d) < 1e-14
        np.testing.assert_allclose(g_d, want, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(g_k, want, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("kind", KINDS)
def test_dense_grad_vs_fd_of_dense_nll(kind):
    """R&W Eq. (5.9) against finite differences of oracle.dense_gp's NLL."""
    w = synth.random_problem(11, 120, kind=kind, p_missing=0.25)
    c = w.components[0]
    nll, g = og.dense_nll_grad(kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)

    def f(j, x):
        th = [math.log(c.variance), math.log(c.lengthscale), math.log(w.noise_var)]
        th[j] = x
        comp = synth.Component(kind, math.exp(th[0]), math.exp(th[1]))
        return dense_gp(lambda tau: ossm.kernel_value(comp, tau), w.t, w.y, w.mask, math.exp(th[2]))[2]

    assert abs(nll - f(0, math.log(c.variance))) < 1e-11 * abs(nll)
    th0 = [math.log(c.variance), math.log(c.lengthscale), math.log(w.noise_var)]
    fd = np.array([richardson(lambda x, j=j: f(j, x), th0[j], 1e-3) for j in range(3)])
    np.testing.assert_allclose(g, fd, rtol=1e-7, atol=1e-7)


@pytest.mark.parametrize("kind", KINDS)
def test_kf_nll_matches_c_oracle(kind):
    """The complex-capable numpy filter's NLL (real inputs) equals the C oracle's."""
    w = synth.random_problem(12, 400, kind=kind, p_missing=0.3, ties=3)
    c = w.components[0]
    nll = float(og.kf_nll(kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask))
    ref = oracle.posterior(w)["nll"]
    assert abs(nll - ref) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("kind", KINDS)
def test_kf_complex_step_equals_dense_gradient(kind):
    """Lemma 1: the state-space NLL is the dense GP NLL, so the
    complex-step gradient of the filter equals R&W Eq. (5.9) on the Gram matrix."""
    w = synth.random_problem(13, 300, kind=kind, p_missing=0.3, ties=2)
    c = w.components[0]
    nd, gd = og.dense_nll_grad(kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
    nk, gk = og.kf_nll_grad(kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
    assert abs(nk - nd) <= 1e-10 * abs(nd)
    np.testing.assert_allclose(gk, gd, rtol=1e-8, atol=1e-8 * (1 + np.max(np.abs(gd))))


def test_kf_complex_step_vs_fd_of_c_oracle():
    """Complex step against finite differences of the C oracle NLL (independent code)."""
    kind = "matern52"
    w = synth.random_problem(14, 2000, kind=kind, p_missing=0.2)
    c = w.components[0]
    _, gk = og.kf_nll_grad(kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
    th0 = [math.log(c.variance), math.log(c.lengthscale), math.log(w.noise_var)]

    def f(j, x):
        th = list(th0)
        th[j] = x
        ww = synth.Workload(w.name, [synth.Component(kind, math.exp(th[0]), math.exp(th[1]))], math.exp(th[2]),
                            w.t, w.y, w.mask)
        return oracle.posterior(ww, smooth=False)["nll"]

    fd = np.array([richardson(lambda x, j=j: f(j, x), th0[j], 1e-3) for j in range(3)])
    np.testing.assert_allclose(gk, fd, rtol=1e-6, atol=1e-6)


# ---------------------------------------------------------------- any SSM (NEXT row f1 widened)
GENERAL_MODELS = {
    "rbf4": [synth.Component("rbf", 1.2, 0.7, order=4)],
    "per3+m32": [synth.Component("periodic", 1.5, 1.0, period=0.7, order=3), synth.Component("matern32", 1.0, 2.0)],
    "quasi1": [synth.Component("quasiperiodic", 2.0, 1.0, period=0.5, order=1, mat_lengthscale=3.0, mat_nu2=3)],
    # the paper's CO2 model C_Per x C_Mat + C_Mat, J = 2, d = 14, at time scale 1/52
    "co2_J2": [synth.Component("quasiperiodic", 2.0, 1.0, period=1.0, order=2, mat_lengthscale=5.0, mat_nu2=3),
               synth.Component("matern32", 10.0, 20.0)],
    "rbf3+m12": [synth.Component("rbf", 1.0, 0.5, order=3), synth.Component("matern12", 0.5, 2.0)],
}


def components_at(comps, theta):
    """The kernel spec at log-hyper-parameters theta (oracle.grad.param_names order)."""
    out, i = [], 0
    for c in comps:
        kw = dict(variance=math.exp(theta[i]), lengthscale=math.exp(theta[i + 1]))
        i += 2
        if c.kind in ("periodic", "quasiperiodic"):
            kw["period"] = math.exp(theta[i]); i += 1
        if c.kind == "quasiperiodic":
            kw["mat_lengthscale"] = math.exp(theta[i]); i += 1
        out.append(synth.Component(c.kind, order=c.order, mat_nu2=c.mat_nu2, **{**dict(period=c.period,
                                   mat_lengthscale=c.mat_lengthscale), **kw}))
    return out, math.exp(theta[i])


def _general_problem(name, n=240, seed=21):
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.exponential(0.02, n))
    if name == "co2_J2":
        t = np.arange(n) / 52.0
    y = np.sin(2 * np.pi * t) + 0.3 * np.cos(7 * t) + 0.2 * rng.standard_normal(n)
    mask = (rng.random(n) > 0.15).astype(np.uint8)
    y[mask == 0] = np.nan
    return GENERAL_MODELS[name], 0.05, t, y, mask


def test_ive_series_vs_scipy():
    from scipy import special
    for j in range(0, 9):
        for a in (1e-3, 0.25, 1.0, 4.0, 25.0):
            assert abs(og.ive_series(j, a) - special.ive(j, a)) <= 1e-14 * max(special.ive(j, a), 1e-300) + 1e-300


@pytest.mark.parametrize("name", list(GENERAL_MODELS))
def test_general_ssm_matches_builder(name):
    """The complex-capable construction at the real theta equals oracle.ssm.build."""
    comps = GENERAL_MODELS[name]
    G, W, H, P = og.ssm_cs(comps, og.theta0(comps, 0.1))
    m = ossm.build(comps)
    for a, b in ((G, m.G), (W, m.W), (P, m.Pinf)):
        assert np.max(np.abs(a - b)) <= 1e-13 * max(1.0, np.max(np.abs(b)))
    np.testing.assert_array_equal(H, m.H)


@pytest.mark.parametrize("name", list(GENERAL_MODELS))
def test_general_complex_step_vs_fd_of_c_oracle(name):
    """Complex-step gradient of any SSM against 4th-order finite differences of the C oracle's NLL
    (independent code: oracle.ssm.build at the perturbed hyper-parameters + kalman.c)."""
    comps, r, t, y, mask = _general_problem(name)
    nll, g = og.kf_nll_grad_general(comps, r, t, y, mask)
    th0 = og.theta0(comps, r)
    assert len(og.param_names(comps)) == th0.shape[0] == g.shape[0]

    def f(j, x):
        th = th0.copy()
        th[j] = x
        cs, rr = components_at(comps, th)
        return oracle.posterior(synth.Workload("g", cs, rr, t, y, mask), smooth=False)["nll"]

    assert abs(nll - f(0, th0[0])) <= 1e-10 * abs(nll)
    fd = np.array([richardson(lambda x, j=j: f(j, x), th0[j], 1e-3) for j in range(th0.shape[0])])
    np.testing.assert_allclose(g, fd, rtol=2e-6, atol=2e-6 * (1 + np.max(np.abs(fd))))


def test_general_equals_matern_specific():
    """For one Matern component the general complex step equals kf_nll_grad (3 parameters)."""
    for kind in KINDS:
        w = synth.random_problem(15, 250, kind=kind, p_missing=0.2, ties=2)
        c = w.components[0]
        n1, g1 = og.kf_nll_grad(kind, c.variance, c.lengthscale, w.noise_var, w.t, w.y, w.mask)
        n2, g2 = og.kf_nll_grad_general(w.components, w.noise_var, w.t, w.y, w.mask)
        assert abs(n1 - n2) <= 1e-12 * abs(n1)
        np.testing.assert_allclose(g2, g1, rtol=1e-11, atol=1e-11 * np.max(np.abs(g1)))
