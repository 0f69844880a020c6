"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 CPU implementation of what the PSSGP hot
path computes (sequential Kalman filter + RTS smoother + NLL, PAPER.md
supplement:285-430), plus the paper's element/operator algebra in numpy and a
dense O(N^3) GP used to pin it (Lemma 1).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import this package.  It shares no code with the
CUDA path (paper_2102_09964_b200/) and never imports it.

Pins and their status are listed in DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import ssm as ssm  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/kalman.c -> oracle/liboracle.so (plain gcc, fp64)."""
    src = os.path.join(_HERE, "kalman.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fno-fast-math", "-ffp-contract=off",
                               "-fPIC", "-shared", "-std=c11", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_expm.argtypes = [ctypes.c_int, dp, dp]
        lib.oracle_discretize.argtypes = [ctypes.c_int, dp, dp, ctypes.c_double, dp, dp]
        lib.oracle_kf_rts.argtypes = [ctypes.c_int, dp, dp, dp, dp, ctypes.c_double, ctypes.c_int64,
                                      dp, dp, ctypes.POINTER(ctypes.c_uint8), dp, dp, dp, dp, dp, dp, dp,
                                      ctypes.POINTER(ctypes.c_int64)]
        for f in (lib.oracle_expm, lib.oracle_discretize, lib.oracle_kf_rts):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleError(RuntimeError):
    def __init__(self, status, index):
        super().__init__(f"oracle status {status} at index {index}")
        self.status = status
        self.index = index


def expm(A: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    E = np.empty_like(A)
    st = _load().oracle_expm(A.shape[0], _p(A), _p(E))
    if st:
        raise OracleError(st, -1)
    return E


def discretize(m, dt: float):
    """(F, Q) for one step of length dt (Van Loan)."""
    G = np.ascontiguousarray(m.G, dtype=np.float64)
    W = np.ascontiguousarray(m.W, dtype=np.float64)
    n = G.shape[0]
    F = np.empty((n, n)); Q = np.empty((n, n))
    st = _load().oracle_discretize(n, _p(G), _p(W), float(dt), _p(F), _p(Q))
    if st:
        raise OracleError(st, -1)
    return F, Q


def kf_rts(m, r: float, t, y, mask, smooth: bool = True, moments: bool = False):
    """Sequential KF + RTS + NLL.  Returns dict(mean, var, nll[, xf, Pf, xs, Ps])."""
    t = np.ascontiguousarray(t, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    N = t.shape[0]
    n = m.n
    G = np.ascontiguousarray(m.G, dtype=np.float64)
    W = np.ascontiguousarray(m.W, dtype=np.float64)
    H = np.ascontiguousarray(m.H, dtype=np.float64)
    P = np.ascontiguousarray(m.Pinf, dtype=np.float64)
    out = {}
    mean = np.empty(N) if smooth else None
    var = np.empty(N) if smooth else None
    nll = np.zeros(1)
    xf = Pf = xs = Ps = None
    if moments:
        xf = np.empty((N, n)); Pf = np.empty((N, n, n))
        if smooth:
            xs = np.empty((N, n)); Ps = np.empty((N, n, n))
    idx = ctypes.c_int64(-1)
    st = _load().oracle_kf_rts(n, _p(G), _p(W), _p(H), _p(P), float(r), N, _p(t), _p(y),
                               mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                               _p(mean), _p(var), _p(nll), _p(xf), _p(Pf), _p(xs), _p(Ps),
                               ctypes.byref(idx))
    if st:
        raise OracleError(st, idx.value)
    out["nll"] = float(nll[0])
    if smooth:
        out["mean"] = mean
        out["var"] = var
    if moments:
        out["xf"], out["Pf"] = xf, Pf
        if smooth:
            out["xs"], out["Ps"] = xs, Ps
    return out


def posterior(workload, balance_model: bool = True, **kw):
    """Convenience: build the SSM of a synth.Workload and run kf_rts on it."""
    m = ssm.build(workload.components, balance_model=balance_model)
    return kf_rts(m, workload.noise_var, workload.t, workload.y, workload.mask, **kw)
