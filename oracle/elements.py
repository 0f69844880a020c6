"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's parallel formulation written out step by step in numpy, in the
paper's notation, for the operator-algebra and Prop. 1 / Prop. 2 tests:

  * Filter elements (A, b, C, eta, J):
      missing y, k > 1: (F_{k-1}, 0, Q_{k-1}, 0, 0)      Eq. (6)+(8)
      missing y, k = 1: (0, 0, P_inf, 0, 0)               Eq. (7)+(8)
      observed,  k > 1: S = H Q H^T + R, K = Q H^T S^-1,
                        A = (I - K H) F, b = K y, C = (I - K H) Q,
                        eta = F^T H^T S^-1 y, J = F^T H^T S^-1 H F
      observed,  k = 1: (0, m_1, P_1, 0, 0), (m_1, P_1) = KF update of
                        N(0, P_inf) with y_1        (reading Z1)
  * Filtering operator, PAPER.md:116-121 (solves, never explicit inverses).
  * Smoother elements (reading Z2, PAPER.md:446-466 / SPEC.md:337):
      k < N: E_k = G_k = P_k F_k^T (F_k P_k F_k^T + Q_k)^-1,
             g_k = xbar_k - E_k F_k xbar_k, L_k = P_k - E_k F_k P_k;
      k = N: (0, xbar_N, P_N).
  * Smoothing operator (E_i, g_i, L_i) (x) (E_j, g_j, L_j)
      = (E_i E_j, E_i g_j + g_i, E_i L_j E_i^T + L_i), i earlier.
  * Prefix scans: sequential left fold (the grouping of the proof)
    and an explicit up-sweep/down-sweep tree (Blelloch).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np

FElem = Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray, np.ndarray]
SElem = Tuple[np.ndarray, np.ndarray, np.ndarray]


def filter_identity(n: int) -> FElem:
    return (np.eye(n), np.zeros(n), np.zeros((n, n)), np.zeros(n), np.zeros((n, n)))


def smoother_identity(n: int) -> SElem:
    return (np.eye(n), np.zeros(n), np.zeros((n, n)))


def filter_combine(ei: FElem, ej: FElem) -> FElem:
    """(A,b,C,eta,J)_i (x) (A,b,C,eta,J)_j."""
    Ai, bi, Ci, ei_, Ji = ei
    Aj, bj, Cj, ej_, Jj = ej
    n = Ai.shape[0]
    I = np.eye(n)
    M = I + Ci @ Jj                     # (I + C_i J_j)
    MT = I + Jj @ Ci                    # (I + J_j C_i)
    A = Aj @ np.linalg.solve(M, Ai)
    b = Aj @ np.linalg.solve(M, bi + Ci @ ej_) + bj
    C = Aj @ np.linalg.solve(M, Ci) @ Aj.T + Cj
    eta = Ai.T @ np.linalg.solve(MT, ej_ - Jj @ bi) + ei_
    J = Ai.T @ np.linalg.solve(MT, Jj) @ Ai + Ji
    return (A, b, C, eta, J)


def smoother_combine(ei: SElem, ej: SElem) -> SElem:
    """(E,g,L)_i (x) (E,g,L)_j, i earlier in time."""
    Ei, gi, Li = ei
    Ej, gj, Lj = ej
    return (Ei @ Ej, Ei @ gj + gi, Ei @ Lj @ Ei.T + Li)


def filter_elements(F: Sequence[np.ndarray], Q: Sequence[np.ndarray], H: np.ndarray,
                    Pinf: np.ndarray, r: float, y: np.ndarray, mask: np.ndarray) -> List[FElem]:
    """F[k], Q[k] = transition INTO step k (k >= 1; F[0], Q[0] unused)."""
    n = Pinf.shape[0]
    h = H.reshape(1, n)
    out = []
    for k in range(len(mask)):
        if k == 0:
            if mask[k]:
                S = float((h @ Pinf @ h.T)[0, 0]) + r
                K = (Pinf @ h.T).reshape(n) / S
                m1 = K * y[k]
                P1 = Pinf - np.outer(K, K) * S
                out.append((np.zeros((n, n)), m1, P1, np.zeros(n), np.zeros((n, n))))
            else:
                out.append((np.zeros((n, n)), np.zeros(n), Pinf.copy(), np.zeros(n), np.zeros((n, n))))
            continue
        Fk, Qk = F[k], Q[k]
        if not mask[k]:
            out.append((Fk.copy(), np.zeros(n), Qk.copy(), np.zeros(n), np.zeros((n, n))))
            continue
        S = float((h @ Qk @ h.T)[0, 0]) + r
        K = (Qk @ h.T).reshape(n) / S
        IKH = np.eye(n) - np.outer(K, h.reshape(n))
        A = IKH @ Fk
        b = K * y[k]
        C = IKH @ Qk
        u = (Fk.T @ h.T).reshape(n)
        eta = u * (y[k] / S)
        J = np.outer(u, u) / S
        out.append((A, b, C, eta, J))
    return out


def smoother_elements(F: Sequence[np.ndarray], Q: Sequence[np.ndarray], xf: np.ndarray,
                      Pf: np.ndarray) -> List[SElem]:
    """Smoother elements from filter output; F[k+1], Q[k+1] map step k -> k+1."""
    N, n = xf.shape
    out = []
    for k in range(N):
        if k == N - 1:
            out.append((np.zeros((n, n)), xf[k].copy(), Pf[k].copy()))
            continue
        Fn, Qn = F[k + 1], Q[k + 1]
        Pm = Fn @ Pf[k] @ Fn.T + Qn
        E = np.linalg.solve(Pm, Fn @ Pf[k]).T         # P_k F^T (P-)^-1
        g = xf[k] - E @ Fn @ xf[k]
        L = Pf[k] - E @ Fn @ Pf[k]
        out.append((E, g, L))
    return out


def sequential_scan(elems: Sequence, op: Callable, reverse: bool = False) -> list:
    """Inclusive prefix (or suffix when reverse) by the sequential grouping of PAPER.md:326-330, 431-435."""
    n = len(elems)
    out = [None] * n
    if n == 0:
        return out
    if not reverse:
        acc = elems[0]
        out[0] = acc
        for k in range(1, n):
            acc = op(acc, elems[k])
            out[k] = acc
    else:
        acc = elems[-1]
        out[-1] = acc
        for k in range(n - 2, -1, -1):
            acc = op(elems[k], acc)
            out[k] = acc
    return out


def tree_scan(elems: Sequence, op: Callable, identity, reverse: bool = False) -> list:
    """Work-efficient up-sweep / down-sweep (Blelloch) inclusive scan, padded
    with the identity element to a power of two."""
    if reverse:
        rev = tree_scan(list(elems)[::-1], lambda a, b: op(b, a), identity, False)
        return rev[::-1]
    n = len(elems)
    if n == 0:
        return []
    m = 1
    while m < n:
        m *= 2
    a = list(elems) + [identity] * (m - n)
    # up-sweep
    d = 1
    while d < m:
        for i in range(2 * d - 1, m, 2 * d):
            a[i] = op(a[i - d], a[i])
        d *= 2
    # down-sweep (exclusive), then convert to inclusive
    a[m - 1] = identity
    d = m // 2
    while d >= 1:
        for i in range(2 * d - 1, m, 2 * d):
            t = a[i - d]
            a[i - d] = a[i]
            a[i] = op(a[i], t)
        d //= 2
    return [op(a[i], elems[i]) for i in range(n)]
