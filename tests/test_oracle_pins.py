"""Pins for the CPU oracle (oracle/): checks against what the paper and the
mathematics fix — never against the oracle's own formulas re-typed.

  * Lemma 1 / Corollary: Kalman smoother
    f-posterior and predictive-decomposition NLL == dense O(N^3) GP.
  * Matern closed forms evaluated in
    50-digit mpmath, vs the oracle's Van Loan discretisation.
  * expm special cases, stationarity F P F^T + Q = P_inf
    (SPEC.md:210), semigroup, Simpson quadrature of the Q
    integral.
  * SPEC hand examples (tests/golden/spec_hand_cases.json, each cited).
  * Invariants: all-missing -> prior, interleaving missing
    points leaves the posterior at observed times and the NLL unchanged
    (SPEC.md:366-367, 460), balancing invariance (Eq. (9)),
    Loewner order Ps <= P.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
import synth
from oracle import dense_gp, ssm

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_cases.json")))


def rel_err(a, b):
    """Normwise mean error / elementwise var error (SURVEY.md §8(c) reading Z14)."""
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def var_err(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


# ---------------------------------------------------------------------------------- Lemma 1
@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
@pytest.mark.parametrize("ell", [0.5, 1.0])
def test_lemma1_config1_grid(kind, ell):
    """Config-1-shaped grid (1000 train + 200 test equally spaced on (0,4))."""
    w = synth.config1()
    comp = synth.Component(kind, 1.0, ell)
    m = ssm.build([comp])
    o = oracle.kf_rts(m, w.noise_var, w.t, w.y, w.mask)
    mean, var, nll = dense_gp.dense_gp(lambda tau: ssm.kernel_value(comp, tau), w.t, w.y, w.mask, w.noise_var)
    assert rel_err(o["mean"], mean) < 1e-9
    assert var_err(o["var"], var) < 1e-9
    assert abs(o["nll"] - nll) / abs(nll) < 1e-9


@pytest.mark.parametrize("seed", range(6))
def test_lemma1_random(seed):
    """Random irregular grids with exact ties (dt = 0), random missing pattern."""
    kind = ["matern12", "matern32", "matern52"][seed % 3]
    w = synth.random_problem(seed, 300, kind=kind, p_missing=0.3, ties=5)
    comp = w.components[0]
    o = oracle.posterior(w)
    mean, var, nll = dense_gp.dense_gp(lambda tau: ssm.kernel_value(comp, tau), w.t, w.y, w.mask, w.noise_var)
    assert rel_err(o["mean"], mean) < 1e-9
    assert var_err(o["var"], var) < 1e-9
    assert abs(o["nll"] - nll) / abs(nll) < 1e-9


@pytest.mark.parametrize("order", [4, 6])
def test_lemma1_rbf_ssm_kernel(order):
    """RBF-Taylor SSM (definition unpinned by the paper, reading Z7) is pinned to
    'the stated construction' through the SSM-implied kernel H e^{G|tau|} P H^T."""
    w = synth.random_problem(7, 120, kind="rbf", p_missing=0.2, lengthscale=0.5, variance=1.0)
    comps = [synth.Component("rbf", 1.0, 0.5, order=order)]
    m = ssm.build(comps)
    o = oracle.kf_rts(m, w.noise_var, w.t, w.y, w.mask)
    # evaluate the SSM-implied kernel exactly on every pairwise lag of the grid
    lags = np.abs(w.t[:, None] - w.t[None, :])
    uniq = np.unique(lags)
    kv = ssm.ssm_kernel(m, uniq)

    def kf(tau):
        tau = np.abs(np.asarray(tau))
        if tau.ndim == 1 and tau.shape[0] == 1 and tau[0] == 0.0:
            return ssm.ssm_kernel(m, tau)
        return kv[np.searchsorted(uniq, tau)]
    mean, var, nll = dense_gp.dense_gp(kf, w.t, w.y, w.mask, w.noise_var)
    assert rel_err(o["mean"], mean) < 1e-8
    assert var_err(o["var"], var) < 1e-8
    assert abs(o["nll"] - nll) / abs(nll) < 1e-9


# ---------------------------------------------------------------------------------- SSM
def test_matern_pinf_closed_form():
    """Unbalanced P_inf equals the closed forms of SURVEY.md §8(c) step 1 (sympy, A.0)."""
    s2, ell = 1.7, 0.8
    lam = math.sqrt(3) / ell
    m = ssm.matern(3, s2, ell)
    np.testing.assert_allclose(m.Pinf, np.diag([s2, lam ** 2 * s2]), rtol=1e-12, atol=1e-12)
    lam = math.sqrt(5) / ell
    k = lam ** 2 * s2 / 3
    m = ssm.matern(5, s2, ell)
    np.testing.assert_allclose(m.Pinf, [[s2, 0, -k], [0, k, 0], [-k, 0, lam ** 4 * s2]], rtol=1e-12, atol=1e-10)
    m = ssm.matern(1, s2, ell)
    np.testing.assert_allclose(m.Pinf, [[s2]], rtol=1e-14)


@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
def test_matern_reconstruction(kind):
    """|H e^{G tau} P_inf H^T - C(tau)| small on tau in [0, 5 ell]."""
    comp = synth.Component(kind, 1.3, 0.7)
    for bal in (False, True):
        m = ssm.build([comp], balance_model=bal)
        taus = np.linspace(0, 5 * 0.7, 50)
        np.testing.assert_allclose(ssm.ssm_kernel(m, taus), ssm.kernel_value(comp, taus), atol=1e-12 * 1.3)


def test_rbf_reconstruction_and_coefficients():
    """RBF order 4/6/8 sup error (1.7e-2 / 3.0e-3 / 6.0e-4) and the
    order-6, ell=1 spectral factor printed in SURVEY.md A.9."""
    taus = np.linspace(0, 5.0, 200)
    errs = []
    for order in (4, 6, 8):
        comp = synth.Component("rbf", 1.0, 1.0, order=order)
        m = ssm.build([comp])
        errs.append(np.max(np.abs(ssm.ssm_kernel(m, taus) - ssm.kernel_value(comp, taus))))
    assert errs[0] > errs[1] > errs[2]          # SPEC.md:145 monotone in order
    assert abs(errs[1] - 3.0e-3) < 0.3e-3
    m = ssm.rbf_taylor(6, 1.0, 1.0)
    a = -m.G[-1, :]
    np.testing.assert_allclose(a[::-1], [11.99887, 65.98646, 210.18825, 404.91535, 443.71196, 214.66253], rtol=2e-6)
    assert abs(m.q - 115505.43) < 0.05


def test_rbf_spectral_factor_vs_mpmath_golden():
    """The oracle's fp64 spectral factor (numpy.roots) and q against the 50-digit construction of
    reading Z7 written independently by tools/gen_rbf_pins.py (tests/golden/rbf_taylor_pins.json)."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rbf_taylor_pins.json")))
    for c in gold["cases"]:
        m = ssm.rbf_taylor(c["order"], c["variance"], c["lengthscale"])
        a = -m.G[-1, :][::-1]                       # companion last row = -(a_0 .. a_{n-1}), low to high
        ref = np.array([float(x) for x in c["a_monic_high_to_low"][1:]])
        np.testing.assert_allclose(a, ref, rtol=1e-11)
        assert abs(m.q - float(c["q"])) <= 1e-13 * float(c["q"])


def test_periodic_reconstruction():
    """Periodic J=6, ell=1: Bessel construction error ~1.3e-6."""
    comp = synth.Component("periodic", 1.0, 1.0, period=1.0, order=6)
    m = ssm.build([comp])
    taus = np.linspace(0, 3.0, 301)
    err = np.max(np.abs(ssm.ssm_kernel(m, taus) - ssm.kernel_value(comp, taus)))
    assert err < 5e-6


def test_sum_kernel_reconstruction():
    comps = [synth.Component("periodic", 4.0, 1.0, period=1.0, order=6), synth.Component("matern32", 10.0, 20.0)]
    m = ssm.build(comps)
    assert m.n == 16
    taus = np.linspace(0, 3.0, 61)
    exact = ssm.kernel_value(comps[0], taus) + ssm.kernel_value(comps[1], taus)
    np.testing.assert_allclose(ssm.ssm_kernel(m, taus), exact, atol=4.0 * 5e-6)


def test_lyapunov_residual():
    rng = np.random.default_rng(0)
    for n in (2, 3, 5):
        A = rng.standard_normal((n, n))
        G = A - (np.max(np.real(np.linalg.eigvals(A))) + 1.0) * np.eye(n)
        P = ssm.lyapunov_vec(G, np.eye(n))
        assert np.max(np.abs(G @ P + P @ G.T + np.eye(n))) < 1e-10
        assert np.min(np.linalg.eigvalsh(P)) > -1e-10


# ---------------------------------------------------------------------------------- expm / discretisation
def test_expm_special_cases():
    np.testing.assert_array_equal(oracle.expm(np.zeros((2, 2))), np.eye(2))
    np.testing.assert_allclose(oracle.expm(np.diag([1.0, 2.0])), np.diag([math.e, math.e ** 2]), rtol=1e-14)
    A = np.array([[0.0, 1.0], [-3.0, -2.0 * math.sqrt(3.0)]]) * 0.5
    T = np.eye(2); term = np.eye(2)
    for k in range(1, 31):
        term = term @ A / k
        T = T + term
    np.testing.assert_allclose(oracle.expm(A), T, rtol=1e-10, atol=1e-12)
    rng = np.random.default_rng(3)
    for n in (3, 8):
        B = rng.standard_normal((n, n)) - 2 * np.eye(n)
        np.testing.assert_allclose(oracle.expm(B) @ oracle.expm(-B), np.eye(n), atol=1e-10)


def _m52_closed_mp(lam, s2, dt):
    """Matern-5/2 F, Q closed forms, 50-digit arithmetic."""
    mp.mp.dps = 50
    lam = mp.mpf(lam); s2 = mp.mpf(s2); D = mp.mpf(dt)
    z = lam * D; e = mp.e ** (-z); x = 2 * z; ex = mp.e ** (-x)
    F = [[e * (1 + z + z ** 2 / 2), e * D * (1 + z), e * D ** 2 / 2],
         [-e * lam ** 3 * D ** 2 / 2, e * (1 + z - z ** 2), e * D * (2 - z) / 2],
         [e * lam ** 3 * D * (z - 2) / 2, e * lam ** 2 * D * (z - 3), e * (1 - 2 * z + z ** 2 / 2)]]
    Q00 = s2 * ex * (mp.e ** x - 1 - x - x ** 2 / 2 - x ** 3 / 6 - x ** 4 / 24)
    Q01 = lam * s2 * ex * x ** 4 / 24
    Q02 = -(lam ** 2 * s2 / 24) * ex * (x ** 4 - 4 * x ** 3 - 4 * x ** 2 - 8 * x + 8 * mp.e ** x - 8)
    Q11 = -(lam ** 2 * s2 / 24) * ex * (x ** 4 - 4 * x ** 3 + 4 * x ** 2 + 8 * x - 8 * mp.e ** x + 8)
    Q12 = (lam ** 3 * s2 / 24) * ex * x ** 2 * (x - 4) ** 2
    Q22 = -(lam ** 4 * s2 / 24) * ex * (x ** 4 - 12 * x ** 3 + 44 * x ** 2 - 40 * x - 24 * mp.e ** x + 24)
    Q = [[Q00, Q01, Q02], [Q01, Q11, Q12], [Q02, Q12, Q22]]
    return np.array(F, dtype=float), np.array(Q, dtype=float)


def _m32_closed_mp(lam, s2, dt):
    mp.mp.dps = 50
    lam = mp.mpf(lam); s2 = mp.mpf(s2); D = mp.mpf(dt)
    z = lam * D; e = mp.e ** (-z); x = 2 * z; ex = mp.e ** (-x)
    F = [[e * (1 + z), e * D], [-e * lam ** 2 * D, e * (1 - z)]]
    Q00 = s2 * ex * (mp.e ** x - 1 - x - x ** 2 / 2)
    Q01 = lam * s2 * ex * x ** 2 / 2
    Q11 = lam ** 2 * s2 * ex * (mp.e ** x - 1 + x - x ** 2 / 2)
    return np.array(F, dtype=float), np.array([[Q00, Q01], [Q01, Q11]], dtype=float)


@pytest.mark.parametrize("dt", [2.4e-7, 1.2e-4, 1e-3, 0.05, 0.3, 1.0, 3.0, 10.0])
@pytest.mark.parametrize("nu2", [3, 5])
def test_discretize_vs_closed_form(nu2, dt):
    ell, s2 = 0.5, 1.3
    m = ssm.matern(nu2, s2, ell)
    lam = math.sqrt(nu2) / ell
    F, Q = oracle.discretize(m, dt)
    Fc, Qc = (_m52_closed_mp if nu2 == 5 else _m32_closed_mp)(lam, s2, dt)
    assert np.max(np.abs(F - Fc)) <= 1e-12 * max(1.0, np.max(np.abs(Fc)))
    assert np.max(np.abs(Q - Qc)) <= 1e-12 * np.max(np.abs(Qc))
    big = np.abs(Qc) > 1e-6 * np.max(np.abs(Qc))
    assert np.max(np.abs(Q - Qc)[big] / np.abs(Qc)[big]) < 1e-9


@pytest.mark.parametrize("kind", ["matern32", "matern52", "rbf"])
def test_discretize_stationarity_semigroup(kind):
    comp = synth.Component(kind, 1.0, 0.5, order=6)
    m = ssm.build([comp])
    for dt in (1e-4, 0.01, 0.3, 2.0):
        F, Q = oracle.discretize(m, dt)
        np.testing.assert_allclose(F @ m.Pinf @ F.T + Q, m.Pinf, atol=1e-10 * np.max(np.abs(m.Pinf)))
        F1, Q1 = oracle.discretize(m, 0.4 * dt)
        F2, Q2 = oracle.discretize(m, 0.6 * dt)
        np.testing.assert_allclose(F2 @ F1, F, atol=1e-10 * max(1.0, np.max(np.abs(F))))
        np.testing.assert_allclose(F2 @ Q1 @ F2.T + Q2, Q, atol=1e-10 * np.max(np.abs(m.Pinf)))
    F0, Q0 = oracle.discretize(m, 0.0)
    np.testing.assert_array_equal(F0, np.eye(m.n))
    np.testing.assert_array_equal(Q0, np.zeros((m.n, m.n)))


def test_discretize_simpson_quadrature():
    """Q equals a composite-Simpson quadrature of the supplement integral."""
    from scipy.linalg import expm
    m = ssm.matern(3, 1.0, 1.0)
    dt = 0.3
    F, Q = oracle.discretize(m, dt)
    s = np.linspace(0, dt, 2001)
    vals = np.array([expm(m.G * (dt - u)) @ m.W @ expm(m.G * (dt - u)).T for u in s])
    w = np.ones(s.shape[0]); w[1:-1:2] = 4; w[2:-1:2] = 2
    Qs = (dt / (s.shape[0] - 1) / 3) * np.einsum("k,kij->ij", w, vals)
    np.testing.assert_allclose(Q, Qs, rtol=1e-10, atol=1e-13)


# ---------------------------------------------------------------------------------- hand cases
def test_spec_one_kf_step_and_nll():
    g = GOLD["one_kf_step"]
    m = ssm.SSM(np.array([[-1.0]]), np.array([[1.0]]), 2.0, np.array([1.0]), np.array([[g["P0"]]]))
    o = oracle.kf_rts(m, g["R"], np.array([0.0]), np.array([g["y"]]), np.array([1], np.uint8), moments=True)
    assert o["xf"][0, 0] == pytest.approx(g["expect"]["x"], abs=1e-15)
    assert o["Pf"][0, 0, 0] == pytest.approx(g["expect"]["P"], abs=1e-15)
    h = GOLD["single_point_lml"]
    m = ssm.matern(1, h["variance"], h["lengthscale"])
    o = oracle.kf_rts(m, h["r"], np.array([0.3]), np.array([h["y"]]), np.array([1], np.uint8))
    assert o["nll"] == pytest.approx(h["expect_nll"], rel=1e-15)
    v = GOLD["single_point_var"]
    m = ssm.matern(3, v["variance"], v["lengthscale"])
    o = oracle.kf_rts(m, v["r"], np.array([1.0]), np.array([0.4]), np.array([1], np.uint8))
    s2, r = v["variance"], v["r"]
    assert o["var"][0] == pytest.approx(s2 * r / (s2 + r), rel=1e-14)


def test_sinusoid_fixture():
    g = GOLD["sinusoid_half"]
    assert abs(synth.sinusoid(np.array([g["t"]]))[0] - g["expect_f"]) < 1e-15


# ---------------------------------------------------------------------------------- invariants
def test_all_missing_is_prior():
    w = synth.random_problem(3, 200, kind="matern52", p_missing=1.0)
    assert w.mask.sum() == 0
    o = oracle.posterior(w)
    assert np.max(np.abs(o["mean"])) == 0.0
    np.testing.assert_allclose(o["var"], w.components[0].variance, rtol=1e-12)
    assert o["nll"] == 0.0


@pytest.mark.parametrize("kind", ["matern32", "matern52"])
def test_interleaving_missing_points(kind):
    """inserting unobserved times changes nothing at observed times."""
    w = synth.random_problem(11, 400, kind=kind, p_missing=0.0)
    base = oracle.posterior(w)
    rng = np.random.default_rng(5)
    t_new = np.sort(rng.uniform(w.t[0] - 0.5, w.t[-1] + 0.5, 250))
    t, mask, order = synth.merged_grid(w.t, t_new)
    y = np.concatenate([w.y, np.full(250, np.nan)])[order]
    w2 = synth.Workload("interleaved", w.components, w.noise_var, t, y, mask)
    o = oracle.posterior(w2)
    obs = mask == 1
    assert rel_err(o["mean"][obs], base["mean"]) < 1e-10
    assert var_err(o["var"][obs], base["var"]) < 1e-10
    assert abs(o["nll"] - base["nll"]) < 1e-10 * abs(base["nll"])


def test_balancing_invariance():
    """Eq. (9): f-posterior and NLL independent of the diagonal scaling D."""
    for kind in ("matern32", "matern52"):
        w = synth.random_problem(21, 300, kind=kind)
        a = oracle.posterior(w, balance_model=True)
        b = oracle.posterior(w, balance_model=False)
        assert rel_err(a["mean"], b["mean"]) < 1e-9
        assert var_err(a["var"], b["var"]) < 1e-9
        assert abs(a["nll"] - b["nll"]) < 1e-9 * abs(b["nll"])


def test_smoothed_cov_below_filtered():
    w = synth.random_problem(4, 200, kind="matern52")
    o = oracle.posterior(w, moments=True)
    for k in range(0, 200, 7):
        ev = np.linalg.eigvalsh(o["Pf"][k] - o["Ps"][k])
        assert ev.min() > -1e-9 * np.max(np.abs(o["Pf"][k]))


def test_input_errors():
    w = synth.random_problem(2, 50)
    t = w.t.copy(); t[20] = t[19] - 1e-3
    with pytest.raises(oracle.OracleError) as e:
        oracle.kf_rts(ssm.build(w.components), w.noise_var, t, w.y, w.mask)
    assert e.value.status == 2 and e.value.index == 20


def test_quasiperiodic_kronecker_reconstruction():
    """Quasi-periodic product: the Kronecker SSM reproduces
    k_per(tau) * k_mat(tau) up to the periodic truncation, and n_x = 10 / 14 / 18 for the
    CO2 model C_Per x C_Mat + C_Mat with J = 1 / 2 / 3."""
    for J, nx in [(1, 10), (2, 14), (3, 18)]:
        w = synth.co2_product(n=10, order=J)
        m = ssm.build(w.components)
        assert m.n == nx
    comp = synth.Component("quasiperiodic", 2.0, 1.0, period=1.0, order=8, mat_lengthscale=3.0, mat_nu2=3)
    m = ssm.build([comp])
    taus = np.linspace(0, 4.0, 81)
    np.testing.assert_allclose(ssm.ssm_kernel(m, taus), ssm.kernel_value(comp, taus), atol=2.0 * 1e-7)
    # stationarity of the product model: G P + P G^T + W = 0
    assert np.max(np.abs(m.G @ m.Pinf + m.Pinf @ m.G.T + m.W)) < 1e-12 * np.max(np.abs(m.W))


def test_lemma1_quasiperiodic_ssm_kernel():
    """Dense GP with the SSM-implied kernel pins the oracle on the product model."""
    w = synth.co2_product(n=400, order=1)
    m = ssm.build(w.components)
    o = oracle.kf_rts(m, w.noise_var, w.t, w.y, w.mask)
    lags = np.unique(np.abs(w.t[:, None] - w.t[None, :]))
    kv = ssm.ssm_kernel(m, lags)

    def kf(tau):
        tau = np.abs(np.asarray(tau))
        if tau.ndim == 1 and tau.shape[0] == 1 and tau[0] == 0.0:
            return ssm.ssm_kernel(m, tau)
        return kv[np.searchsorted(lags, tau)]
    mean, var, nll = dense_gp.dense_gp(kf, w.t, w.y, w.mask, w.noise_var)
    assert rel_err(o["mean"], mean) < 1e-8
    assert var_err(o["var"], var) < 1e-8
    assert abs(o["nll"] - nll) / abs(nll) < 1e-9
