"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Continuous state-space models (G, L, q, H, P_inf) of the covariance functions
the hot path supports, built in plain numpy/scipy, independently of the
library's C++ model builder.

  * Eq. (2): dx/dt = G x + L w, y_k = H x(t_k) + e_k, w white
    with spectral density q; Matern closed forms are exact.
  * Matern-nu: lambda = sqrt(2 nu)/ell, companion drift,
    q chosen so that H P_inf H^T = sigma^2 (checked against the closed-form
    P_inf of SURVEY.md §8(c) by tests/test_oracle_pins.py::test_matern_pinf_closed_form).
  * RBF Taylor approximation (reading Z7):
    Taylor-expand 1/S(omega) to order n, take the left-half-plane spectral
    factor a(s) (numpy.roots), G = companion(a), L = e_n,
    q = sigma^2 sqrt(2 pi) ell n! (2/ell^2)^n.
  * Periodic kernel as harmonic oscillators (PAPER.md:224, SPEC.md:152,
    reading Z8): blocks [[0, -j w0],[j w0, 0]], j = 0..J, no process noise,
    P_inf_j = q_j^2 I, q_0^2 = s2 I_0(ell^-2) e^{-ell^-2},
    q_j^2 = 2 s2 I_j(ell^-2) e^{-ell^-2}.
  * Sum of kernels: block-diagonal G, P_inf, L q L^T; H concatenated.
  * Stationary covariance by the vectorised Lyapunov solution (§4.1,
    PAPER.md:140-141): (I (x) G + G (x) I) vec P = -vec(L q L^T).
  * Balancing (§4.2 Eq. (9)): Osborne iteration, powers of
    two; balanced model (D^-1 G D, D^-1 L, H D, D^-1 P_inf D^-1) (reading Z5).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy import special


@dataclass
class SSM:
    G: np.ndarray      # n x n drift
    L: np.ndarray      # n x 1 noise loading
    q: float           # white-noise spectral density (scalar)
    H: np.ndarray      # (n,) observation row
    Pinf: np.ndarray   # n x n stationary covariance
    Wmat: object = None  # explicit L q L^T (sums of kernels), else derived from L, q

    @property
    def n(self) -> int:
        return self.G.shape[0]

    @property
    def W(self) -> np.ndarray:
        """L q L^T."""
        if self.Wmat is not None:
            return self.Wmat
        return self.q * (self.L @ self.L.T)


def lyapunov_vec(G: np.ndarray, W: np.ndarray) -> np.ndarray:
    """§4.1: solve G P + P G^T + W = 0 by vectorisation."""
    n = G.shape[0]
    I = np.eye(n)
    K = np.kron(I, G) + np.kron(G, I)
    P = np.linalg.solve(K, -W.reshape(-1)).reshape(n, n)
    return 0.5 * (P + P.T)


def matern(nu2: int, variance: float, lengthscale: float) -> SSM:
    """Matern-nu with nu = nu2/2 in {1/2, 3/2, 5/2}."""
    if nu2 == 1:
        lam = 1.0 / lengthscale
        G = np.array([[-lam]])
        q = 2.0 * variance * lam
    elif nu2 == 3:
        lam = math.sqrt(3.0) / lengthscale
        G = np.array([[0.0, 1.0], [-lam ** 2, -2.0 * lam]])
        q = 4.0 * variance * lam ** 3
    elif nu2 == 5:
        lam = math.sqrt(5.0) / lengthscale
        G = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [-lam ** 3, -3.0 * lam ** 2, -3.0 * lam]])
        q = 16.0 / 3.0 * variance * lam ** 5
    else:
        raise ValueError(nu2)
    n = G.shape[0]
    L = np.zeros((n, 1)); L[-1, 0] = 1.0
    H = np.zeros(n); H[0] = 1.0
    Pinf = lyapunov_vec(G, q * (L @ L.T))
    return SSM(G, L, q, H, Pinf)


def rbf_taylor(order: int, variance: float, lengthscale: float) -> SSM:
    """RBF via Taylor expansion of 1/S(omega)."""
    n = order
    ell2 = lengthscale ** 2
    # P(s) = sum_j (ell^2/2)^j (-s^2)^j / j!  (coefficients in s, highest power first)
    coeffs = np.zeros(2 * n + 1)
    for j in range(n + 1):
        coeffs[2 * n - 2 * j] = (ell2 / 2.0) ** j * (-1.0) ** j / math.factorial(j)
    roots = np.roots(coeffs)
    lhp = roots[roots.real < 0]
    if lhp.shape[0] != n:
        raise ValueError("spectral factorisation failed")
    a = np.real(np.poly(lhp))          # monic, highest power first: s^n + a_{n-1} s^{n-1} + ...
    G = np.zeros((n, n))
    G[:-1, 1:] = np.eye(n - 1)
    G[-1, :] = -a[::-1][:n]            # -[a0, a1, ..., a_{n-1}]
    L = np.zeros((n, 1)); L[-1, 0] = 1.0
    H = np.zeros(n); H[0] = 1.0
    q = variance * math.sqrt(2.0 * math.pi) * lengthscale * math.factorial(n) * (2.0 / ell2) ** n
    return SSM(G, L, q, H, np.zeros((n, n)))   # P_inf filled after balancing


def periodic(J: int, variance: float, lengthscale: float, period: float) -> SSM:
    """Harmonic-oscillator expansion of the periodic kernel (reading Z8)."""
    w0 = 2.0 * math.pi / period
    n = 2 * (J + 1)
    G = np.zeros((n, n)); Pinf = np.zeros((n, n)); H = np.zeros(n)
    a = lengthscale ** -2
    for j in range(J + 1):
        G[2 * j, 2 * j + 1] = -j * w0
        G[2 * j + 1, 2 * j] = j * w0
        qj2 = (1.0 if j == 0 else 2.0) * variance * special.ive(j, a)   # ive = I_j(a) e^{-a}
        Pinf[2 * j, 2 * j] = Pinf[2 * j + 1, 2 * j + 1] = qj2
        H[2 * j] = 1.0
    return SSM(G, np.zeros((n, 1)), 0.0, H, Pinf)


def quasiperiodic(J: int, variance: float, lengthscale: float, period: float, mat_nu2: int,
                  mat_lengthscale: float) -> SSM:
    """Product C_per(tau) C_mat(tau): Kronecker-sum drift
    G = G_p (x) I + I (x) G_m, P_inf = P_p (x) P_m, L q L^T = P_p (x) W_m, H = H_p (x) H_m,
    so that H e^{G tau} P_inf H^T = k_per(tau) k_mat(tau)."""
    per = periodic(J, variance, lengthscale, period)
    mat = matern(mat_nu2, 1.0, mat_lengthscale)
    Ip, Im = np.eye(per.n), np.eye(mat.n)
    G = np.kron(per.G, Im) + np.kron(Ip, mat.G)
    P = np.kron(per.Pinf, mat.Pinf)
    W = np.kron(per.Pinf, mat.W)
    H = np.kron(per.H, mat.H)
    return SSM(G, np.zeros((G.shape[0], 1)), 0.0, H, P, Wmat=W)


def osborne(G: np.ndarray, max_sweeps: int = 100) -> np.ndarray:
    """Osborne balancing with powers of two (reading Z6): returns
    the diagonal of D such that D^-1 G D has comparable off-diagonal row and
    column 1-norms."""
    n = G.shape[0]
    d = np.ones(n)
    A = G.copy()
    for _ in range(max_sweeps):
        changed = False
        for i in range(n):
            c = np.sum(np.abs(A[:, i])) - abs(A[i, i])
            r = np.sum(np.abs(A[i, :])) - abs(A[i, i])
            if c == 0.0 or r == 0.0:
                continue
            f = 1.0
            s = c + r
            while c < r / 2.0:
                c *= 2.0; r /= 2.0; f *= 2.0
            while c >= r * 2.0:
                c /= 2.0; r *= 2.0; f /= 2.0
            if (c + r) < 0.95 * s:
                changed = True
                d[i] *= f
                A[:, i] *= f
                A[i, :] /= f
        if not changed:
            break
    return d


def balance(m: SSM) -> SSM:
    """Eq. (9): z = D^-1 x; (D^-1 G D, D^-1 L, H D, D^-1 P_inf D^-1)."""
    d = osborne(m.G)
    Di = 1.0 / d
    G = (Di[:, None] * m.G) * d[None, :]
    L = Di[:, None] * m.L
    H = m.H * d
    P = (Di[:, None] * m.Pinf) * Di[None, :]
    return SSM(G, L, m.q, H, P)


def block_sum(parts) -> SSM:
    """Sum of kernels: block-diagonal state."""
    n = sum(p.n for p in parts)
    G = np.zeros((n, n)); P = np.zeros((n, n)); W = np.zeros((n, n)); H = np.zeros(n)
    o = 0
    for p in parts:
        k = p.n
        G[o:o + k, o:o + k] = p.G
        P[o:o + k, o:o + k] = p.Pinf
        W[o:o + k, o:o + k] = p.W
        H[o:o + k] = p.H
        o += k
    return SSM(G, np.zeros((n, 1)), 0.0, H, P, Wmat=W)


def build(components, balance_model: bool = True) -> SSM:
    """Kernel spec (list of synth.Component-like objects) -> continuous SSM."""
    parts = []
    for c in components:
        kind = c.kind
        if kind in ("matern12", "matern32", "matern52"):
            m = matern({"matern12": 1, "matern32": 3, "matern52": 5}[kind], c.variance, c.lengthscale)
            if balance_model:
                m = balance(m)
        elif kind == "rbf":
            m = rbf_taylor(c.order, c.variance, c.lengthscale)
            if balance_model:
                m = balance(m)
            m.Pinf = lyapunov_vec(m.G, m.W)
        elif kind == "periodic":
            m = periodic(c.order, c.variance, c.lengthscale, c.period)
        elif kind == "quasiperiodic":
            m = quasiperiodic(c.order, c.variance, c.lengthscale, c.period, c.mat_nu2, c.mat_lengthscale)
        else:
            raise ValueError(kind)
        parts.append(m)
    if len(parts) == 1:
        return parts[0]
    return block_sum(parts)


# ------------------------------------------------------------------ covariance functions
def kernel_value(c, tau: np.ndarray) -> np.ndarray:
    """Exact covariance functions C(tau) (for the dense-GP pin, Lemma 1)."""
    tau = np.abs(np.asarray(tau, dtype=np.float64))
    s2, ell = c.variance, c.lengthscale
    if c.kind == "matern12":
        return s2 * np.exp(-tau / ell)
    if c.kind == "matern32":
        a = math.sqrt(3.0) * tau / ell
        return s2 * (1.0 + a) * np.exp(-a)
    if c.kind == "matern52":
        a = math.sqrt(5.0) * tau / ell
        return s2 * (1.0 + a + a * a / 3.0) * np.exp(-a)
    if c.kind == "rbf":
        return s2 * np.exp(-0.5 * tau ** 2 / ell ** 2)
    if c.kind == "periodic":
        return s2 * np.exp(-2.0 * np.sin(np.pi * tau / c.period) ** 2 / ell ** 2)
    if c.kind == "quasiperiodic":
        per = s2 * np.exp(-2.0 * np.sin(np.pi * tau / c.period) ** 2 / ell ** 2)
        a = math.sqrt(c.mat_nu2) * tau / c.mat_lengthscale
        mat = {1: np.exp(-a), 3: (1.0 + a) * np.exp(-a), 5: (1.0 + a + a * a / 3.0) * np.exp(-a)}[c.mat_nu2]
        return per * mat
    raise ValueError(c.kind)


def ssm_kernel(m: SSM, tau: np.ndarray) -> np.ndarray:
    """SSM-implied covariance k(tau) = H e^{G|tau|} P_inf H^T (Lemma 1 construction)."""
    from scipy.linalg import expm
    tau = np.abs(np.asarray(tau, dtype=np.float64)).reshape(-1)
    out = np.empty_like(tau)
    for i, s in enumerate(tau):
        out[i] = m.H @ expm(m.G * s) @ m.Pinf @ m.H
    return out
