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
