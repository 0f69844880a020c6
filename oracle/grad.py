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


# ---------------------------------------------------------------- any SSM (sums, products), complex step
# The hyper-parameter vector of a kernel spec (the library's order, include/pssgp.h): per component
#   Matern-nu, RBF:   log variance, log lengthscale
#   periodic:         log variance, log lengthscale, log period
#   quasi-periodic:   log variance, log lengthscale, log period, log Matern lengthscale
# then log noise variance.  The SSM is rebuilt at complex hyper-parameters theta + i h e_p with
# constructions made of arithmetic only (so the complex step is exact to rounding): the Bessel
# coefficients by their power series, the RBF spectral factor from the lengthscale-1 factor a_1 by
# a_ell(s) = ell^-n a_1(ell s) (p_ell(s) = p_1(ell s), so the roots are r / ell; no complex roots
# enter the complex step, which would lose it to rounding).  The balancing
# matrix D of the real model is applied unchanged ("D treated as constant").
def param_names(components):
    out = []
    for i, c in enumerate(components):
        out += [f"c{i}.log_variance", f"c{i}.log_lengthscale"]
        if c.kind in ("periodic", "quasiperiodic"):
            out.append(f"c{i}.log_period")
        if c.kind == "quasiperiodic":
            out.append(f"c{i}.log_mat_lengthscale")
    return out + ["log_noise_variance"]


def ive_series(j: int, a):
    """I_j(a) e^{-a} by the power series sum_m (a/2)^(2m+j) / (m! (m+j)!) (Abramowitz & Stegun
    9.6.10); plain arithmetic, so valid for a complex-stepped a."""
    term = 1.0 + 0.0 * a
    for k in range(1, j + 1):
        term = term * (a / 2.0) / k
    total = 0.0 * a
    q = a * a / 4.0
    for m in range(400):
        total = total + term
        term = term * q / ((m + 1.0) * (m + 1.0 + j))
        if abs(term) < 1e-18 * abs(total) and m > abs(a):
            break
    return total * np.exp(-a)


def _rbf_cs(order: int, variance, ell):
    n = order
    coeffs = np.zeros(2 * n + 1)
    for j in range(n + 1):
        coeffs[2 * n - 2 * j] = 0.5 ** j * (-1.0) ** j / math.factorial(j)      # ell = 1
    roots = np.roots(coeffs)
    a1 = np.real(np.poly(roots[roots.real < 0]))            # monic spectral factor at ell = 1
    # roots of p_ell are r / ell, so a_ell(s) = ell^-n a_1(ell s): coefficient of s^k scales by
    # ell^(k - n) (real arithmetic in ell: no complex intermediates for the complex step)
    a = np.array([a1[i] * ell ** (-i) for i in range(n + 1)])   # a1[i] multiplies s^(n - i)
    dtype = np.result_type(a, variance, ell)
    G = np.zeros((n, n), dtype=dtype)
    G[:-1, 1:] = np.eye(n - 1)
    G[-1, :] = -a[::-1][:n]
    q = variance * math.sqrt(2.0 * math.pi) * ell * math.factorial(n) * (2.0 / ell ** 2) ** n
    W = np.zeros((n, n), dtype=dtype)
    W[-1, -1] = q
    return G, W


def _matern_cs(nu2: int, variance, ell):
    dtype = np.result_type(variance, ell, 1.0)
    lam = math.sqrt(nu2) / ell
    n = (nu2 + 1) // 2
    G = np.zeros((n, n), dtype=dtype)
    if n == 1:
        G[0, 0] = -lam
        q = 2.0 * variance * lam
    elif n == 2:
        G[0, 1] = 1.0; G[1, 0] = -lam ** 2; G[1, 1] = -2.0 * lam
        q = 4.0 * variance * lam ** 3
    else:
        G[0, 1] = 1.0; G[1, 2] = 1.0
        G[2, 0] = -lam ** 3; G[2, 1] = -3.0 * lam ** 2; G[2, 2] = -3.0 * lam
        q = 16.0 / 3.0 * variance * lam ** 5
    W = np.zeros((n, n), dtype=dtype)
    W[-1, -1] = q
    return G, W, ssm_mod.lyapunov_vec(G, W)


def _periodic_cs(J: int, variance, ell, period):
    dtype = np.result_type(variance, ell, period, 1.0)
    n = 2 * (J + 1)
    w0 = 2.0 * math.pi / period
    G = np.zeros((n, n), dtype=dtype)
    P = np.zeros((n, n), dtype=dtype)
    a = ell ** -2
    for j in range(J + 1):
        G[2 * j, 2 * j + 1] = -j * w0
        G[2 * j + 1, 2 * j] = j * w0
        P[2 * j, 2 * j] = P[2 * j + 1, 2 * j + 1] = (1.0 if j == 0 else 2.0) * variance * ive_series(j, a)
    return G, P


def ssm_cs(components, theta):
    """(G, W, H, P_inf) at the log-hyper-parameters theta (real or complex), balanced with the D of
    the real model (oracle.ssm.build) held constant."""
    blocks = []
    i = 0
    ex = np.exp
    for c in components:
        s2 = ex(theta[i]); ell = ex(theta[i + 1]); i += 2
        if c.kind in ("matern12", "matern32", "matern52"):
            G, W, P = _matern_cs({"matern12": 1, "matern32": 3, "matern52": 5}[c.kind], s2, ell)
            H = np.zeros(G.shape[0]); H[0] = 1.0
        elif c.kind == "rbf":
            G, W = _rbf_cs(c.order, s2, ell)
            H = np.zeros(G.shape[0]); H[0] = 1.0
            P = None
        elif c.kind == "periodic":
            per = ex(theta[i]); i += 1
            G, P = _periodic_cs(c.order, s2, ell, per)
            W = np.zeros_like(G)
            H = np.zeros(G.shape[0]); H[0::2] = 1.0
        elif c.kind == "quasiperiodic":
            per = ex(theta[i]); mell = ex(theta[i + 1]); i += 2
            Gp, Pp = _periodic_cs(c.order, s2, ell, per)
            Gm, Wm, Pm = _matern_cs(c.mat_nu2, 1.0, mell)
            Ip, Im = np.eye(Gp.shape[0]), np.eye(Gm.shape[0])
            G = np.kron(Gp, Im) + np.kron(Ip, Gm)
            P = np.kron(Pp, Pm)
            W = np.kron(Pp, Wm)
            Hp = np.zeros(Gp.shape[0]); Hp[0::2] = 1.0
            Hm = np.zeros(Gm.shape[0]); Hm[0] = 1.0
            H = np.kron(Hp, Hm)
        else:
            raise ValueError(c.kind)
        if c.kind in ("matern12", "matern32", "matern52", "rbf"):
            # the balancing of oracle.ssm.build, from the real model, held constant
            Gr = np.real(G) if np.iscomplexobj(G) else G
            d = ssm_mod.osborne(Gr)
            Di = 1.0 / d
            G = (Di[:, None] * G) * d[None, :]
            W = (Di[:, None] * W) * Di[None, :]
            H = H * d
            if P is not None:
                P = (Di[:, None] * P) * Di[None, :]
        if P is None:
            P = ssm_mod.lyapunov_vec(G, W)
        blocks.append((G, W, H, P))
    n = sum(b[0].shape[0] for b in blocks)
    dtype = np.result_type(*[b[0] for b in blocks], *[b[1] for b in blocks], *[b[3] for b in blocks])
    G = np.zeros((n, n), dtype=dtype); W = np.zeros((n, n), dtype=dtype); P = np.zeros((n, n), dtype=dtype)
    H = np.zeros(n)
    o = 0
    for g, w, h, p in blocks:
        k = g.shape[0]
        G[o:o + k, o:o + k] = g; W[o:o + k, o:o + k] = w; P[o:o + k, o:o + k] = p; H[o:o + k] = h
        o += k
    return G, W, H, P


def theta0(components, noise_var):
    """The real log-hyper-parameter vector of a kernel spec (param_names order)."""
    th = []
    for c in components:
        th += [math.log(c.variance), math.log(c.lengthscale)]
        if c.kind in ("periodic", "quasiperiodic"):
            th.append(math.log(c.period))
        if c.kind == "quasiperiodic":
            th.append(math.log(c.mat_lengthscale))
    return np.array(th + [math.log(noise_var)])


def kf_nll_theta(components, theta, t, y, mask):
    """Sequential Kalman-filter NLL (supplement PAPER.md:304-315) of the model at theta, in the
    scalar type of theta (complex for the complex step)."""
    G, W, H, P = ssm_cs(components, theta)
    r = np.exp(theta[-1])
    n = G.shape[0]
    dtype = np.result_type(G, W, P, r)
    x = np.zeros(n, dtype=dtype)
    P = P.astype(dtype)
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
            S = H @ P @ H + r
            v = y[k] - H @ x
            Kg = P @ H / S
            nll = nll + 0.5 * (np.log(2.0 * math.pi * S) + v * v / S)
            x = x + Kg * v
            P = P - np.outer(Kg, Kg) * S
            P = 0.5 * (P + P.T)
    return nll


def kf_nll_grad_general(components, noise_var, t, y, mask, h: float = 1e-20):
    """(nll, grad) of the NLL in the log-hyper-parameters (param_names order), complex step."""
    th = theta0(components, noise_var)
    nll = float(np.real(kf_nll_theta(components, th, t, y, mask)))
    grad = np.empty(th.shape[0])
    for p in range(th.shape[0]):
        tc = th.astype(complex)
        tc[p] += 1j * h
        grad[p] = np.imag(kf_nll_theta(components, tc, t, y, mask)) / h
    return nll, grad


def components_at(components, theta):
    """The kernel spec and noise variance at log-hyper-parameters theta (param_names order)."""
    import dataclasses
    out, i = [], 0
    for c in components:
        kw = dict(variance=math.exp(theta[i]), lengthscale=math.exp(theta[i + 1]))
        i += 2
        if c.kind in ("periodic", "quasiperiodic"):
            kw["period"] = math.exp(theta[i]); i += 1
        if c.kind == "quasiperiodic":
            kw["mat_lengthscale"] = math.exp(theta[i]); i += 1
        out.append(dataclasses.replace(c, **kw))
    return out, math.exp(theta[i])
