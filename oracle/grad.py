"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Gradient of the negative log marginal likelihood with respect to
theta = (log sigma^2, log ell, log sigma_n^2) of ONE Matern component — the
hyper-parameter gradient the paper obtains by automatic differentiation of the
(parallel) filter, PAPER.md:77, 157, 173 (NEXT row f1 of SURVEY.md §8).

Two independent definitions, neither shares code with the CUDA path:

* dense_nll_grad — the textbook gradient of the Gaussian log likelihood on the
  dense Gram matrix (Rasmussen & Williams 2006, Eq. (5.9)):
      d NLL / d theta_j = 0.5 tr(K~^-1 dK~_j) - 0.5 alpha^T dK~_j alpha,
      alpha = K~^-1 y,  K~ = K_f(theta) + sigma_n^2 I,
  with dK_f / d log sigma^2 = K_f, dK~ / d log sigma_n^2 = sigma_n^2 I and
  dK_f / d log ell the derivative of the closed-form Matern covariance.  By
  Lemma 1 its NLL is the state-space NLL, so this is also
  the state-space gradient.  O(n^3): small n only.

* kf_nll_grad — the complex-step derivative (Im f(theta + i h) / h, exact to
  rounding for a holomorphic f) of the plain sequential Kalman-filter NLL
  (supplement PAPER.md:304-315; predictive decomposition, reading Z3), with the
  discretisation F = expm(G dt) and Q from the Van Loan block exponential
  evaluated in complex arithmetic.  O(n) with one expm per distinct dt: used for
  grids too large for the dense form.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.linalg import cho_factor, cho_solve, expm

from . import ssm as ssm_mod

_NU2 = {"matern12": 1, "matern32": 3, "matern52": 5}


# ---------------------------------------------------------------- dense (R&W Eq. 5.9)
def matern_k_and_dlogell(nu2: int, s2: float, ell: float, tau: np.ndarray):
    """Closed-form Matern covariance and its derivative in log ell.
    With a = sqrt(nu2) |tau| / ell (da / d log ell = -a):
      nu = 1/2: k = s2 e^-a,                dk = s2 a e^-a
      nu = 3/2: k = s2 (1 + a) e^-a,         dk = s2 a^2 e^-a
      nu = 5/2: k = s2 (1 + a + a^2/3) e^-a, dk = s2 a^2 (1 + a) e^-a / 3."""
    a = math.sqrt(nu2) * np.abs(tau) / ell
    e = np.exp(-a)
    if nu2 == 1:
        return s2 * e, s2 * a * e
    if nu2 == 3:
        return s2 * (1.0 + a) * e, s2 * a * a * e
    if nu2 == 5:
        return s2 * (1.0 + a + a * a / 3.0) * e, s2 * a * a * (1.0 + a) * e / 3.0
    raise ValueError(nu2)


def dense_nll_grad(kind: str, variance: float, lengthscale: float, noise_var: float, t, y, mask):
    """(nll, grad[3]) on the observed points of (t, y, mask) — R&W Eq. (5.9)."""
    obs = np.asarray(mask) != 0
    to = np.asarray(t, dtype=np.float64)[obs]
    yo = np.asarray(y, dtype=np.float64)[obs]
    n = to.shape[0]
    if n == 0:
        return 0.0, np.zeros(3)
    Kf, dKl = matern_k_and_dlogell(_NU2[kind], variance, lengthscale, to[:, None] - to[None, :])
    K = Kf + noise_var * np.eye(n)
    cf = cho_factor(K, lower=True)
    alpha = cho_solve(cf, yo)
    Kinv = cho_solve(cf, np.eye(n))
    nll = 0.5 * (yo @ alpha + 2.0 * np.sum(np.log(np.diag(cf[0]))) + n * math.log(2.0 * math.pi))
    grad = np.empty(3)
    for j, dK in enumerate((Kf, dKl, noise_var * np.eye(n))):
        grad[j] = 0.5 * np.sum(Kinv * dK) - 0.5 * alpha @ dK @ alpha
    return float(nll), grad


# ---------------------------------------------------------------- sequential KF, complex step
def _van_loan(G, W, dt):
    """F = expm(G dt); Q = int_0^dt e^{G s} W e^{G^T s} ds from the block exponential
    expm([[G, W], [0, -G^T]] dt) = [[F, Q F^-T], [0, F^-T]] (Van Loan 1978)."""
    n = G.shape[0]
    C = np.zeros((2 * n, 2 * n), dtype=G.dtype)
    C[:n, :n] = G
    C[:n, n:] = W
    C[n:, n:] = -G.T
    E = expm(C * dt)
    F = E[:n, :n]
    Q = E[:n, n:] @ F.T
    return F, 0.5 * (Q + Q.T)


def kf_nll(kind: str, variance, lengthscale, noise_var, t, y, mask):
    """Plain sequential Kalman-filter NLL (supplement PAPER.md:304-315), arithmetic in
    whatever scalar type the hyper-parameters carry (float or complex)."""
    m = ssm_mod.matern(_NU2[kind], variance, lengthscale)
    G, W, H = m.G, m.W, m.H.astype(np.float64)
    n = G.shape[0]
    dtype = np.result_type(G, W, noise_var)
    x = np.zeros(n, dtype=dtype)
    P = m.Pinf.astype(dtype)
    t = np.asarray(t, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    cache = {}
    nll = dtype.type(0)
    for k in range(t.shape[0]):
        if k > 0:
            dt = t[k] - t[k - 1]
            if dt not in cache:
                cache[dt] = _van_loan(G.astype(dtype), W.astype(dtype), dt)
            F, Q = cache[dt]
            x = F @ x
            P = F @ P @ F.T + Q
        if mask[k]:
            S = H @ P @ H + noise_var
            v = y[k] - H @ x
            Kg = P @ H / S
            nll = nll + 0.5 * (np.log(2.0 * math.pi * S) + v * v / S)
            x = x + Kg * v
            P = P - np.outer(Kg, Kg) * S
            P = 0.5 * (P + P.T)
    return nll


def kf_nll_grad(kind: str, variance: float, lengthscale: float, noise_var: float, t, y, mask, h: float = 1e-20):
    """(nll, grad[3]) by complex-step differentiation of kf_nll in each log-parameter."""
    nll = float(np.real(kf_nll(kind, variance, lengthscale, noise_var, t, y, mask)))
    grad = np.empty(3)
    e = complex(math.cos(h), math.sin(h))  # exp(i h): theta -> theta + i h in log space
    grad[0] = np.imag(kf_nll(kind, variance * e, lengthscale, noise_var, t, y, mask)) / h
    grad[1] = np.imag(kf_nll(kind, variance, lengthscale * e, noise_var, t, y, mask)) / h
    grad[2] = np.imag(kf_nll(kind, variance, lengthscale, noise_var * e, t, y, mask)) / h
    return nll, grad
