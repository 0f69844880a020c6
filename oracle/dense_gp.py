"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Naive O(N^3) GP regression, used only as a
PIN for the sequential oracle through Lemma 1 / Corollary (PAPER.md:262-283,
476-478): for state-space-representable covariances the Kalman smoother's
f-posterior and the predictive-decomposition likelihood equal the dense GP's.

  K~ = K(t_obs, t_obs) + r I  (Cholesky),  mean(t*) = k*^T K~^-1 y,
  var(t*) = C(0) - k*^T K~^-1 k*,
  NLL = 0.5 (y^T K~^-1 y + log|K~| + n log 2 pi).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import cho_factor, cho_solve


def dense_gp(kfun, t: np.ndarray, y: np.ndarray, mask: np.ndarray, r: float):
    """kfun(tau) -> covariance; returns (mean, var, nll) on the whole grid t."""
    obs = mask != 0
    to, yo = t[obs], y[obs]
    n = to.shape[0]
    Kst = kfun(t[:, None] - to[None, :]) if n else np.zeros((t.shape[0], 0))
    k0 = float(kfun(np.array([0.0]))[0])
    if n == 0:
        return np.zeros_like(t), np.full_like(t, k0), 0.0
    K = kfun(to[:, None] - to[None, :]) + r * np.eye(n)
    cf = cho_factor(K, lower=True)
    alpha = cho_solve(cf, yo)
    mean = Kst @ alpha
    V = cho_solve(cf, Kst.T)
    var = k0 - np.einsum("ij,ji->i", Kst, V)
    logdet = 2.0 * np.sum(np.log(np.diag(cf[0])))
    nll = 0.5 * (yo @ alpha + logdet + n * np.log(2.0 * np.pi))
    return mean, var, float(nll)
