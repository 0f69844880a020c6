"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no state-space model, no
discretisation, no filtering): only the input recipes of SURVEY.md §8(d) /
DESIGN.md "Input recipe" — time grids, observation masks and noisy
observations — drawn from numpy PCG64 generators with fixed seeds
(noise seed 0, time-jitter seed 1, mask seed 2).

Paper passages the recipes follow:
  * Eq. (10), PAPER.md:185-191 (§5.1): f(t) = sin(pi t) + sin(2 pi t) + sin(3 pi t),
    observations "equally spaced on (0, 4)"; finest grid 2^15 points on (0,4)
     -> h = 4 / 2^15.
  * §5.3: CO2-like weekly series with a yearly period (config C4).
  * supplement PAPER.md:255: test points are missing observations on the
    sorted merged grid (mask = 0, y ignored; we store NaN there on purpose).

Kernel hyper-parameters of each config are plain data here (SURVEY.md §8(c)
reading Z10: sigma^2 = 1, lengthscale 0.5, sigma_n = 0.1 for the sinusoid).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

H_FINE = 4.0 / 2 ** 15          # PAPER.md:193 densest grid on (0, 4)
SEED_NOISE, SEED_JITTER, SEED_MASK = 0, 1, 2


@dataclass
class Component:
    """One additive covariance component (kind names follow SPEC.md:109)."""
    kind: str                    # 'matern12' | 'matern32' | 'matern52' | 'rbf' | 'periodic' | 'quasiperiodic'
    variance: float = 1.0
    lengthscale: float = 1.0
    period: float = 1.0
    order: int = 0               # RBF Taylor order / periodic harmonics J
    mat_lengthscale: float = 1.0  # quasi-periodic: lengthscale of the Matern factor
    mat_nu2: int = 3             # quasi-periodic: 2 nu of the Matern factor


@dataclass
class Workload:
    name: str
    components: List[Component]
    noise_var: float
    t: np.ndarray                # float64, non-decreasing
    y: np.ndarray                # float64, NaN where mask == 0
    mask: np.ndarray             # uint8, 1 = observed, 0 = missing / test point
    uniform_dt: float = 0.0      # > 0 when every step has exactly this dt
    meta: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return int(self.t.shape[0])


def sinusoid(t: np.ndarray) -> np.ndarray:
    """Eq. (10)."""
    return np.sin(np.pi * t) + np.sin(2 * np.pi * t) + np.sin(3 * np.pi * t)


def _noisy(f: np.ndarray, sigma: float, seed: int = SEED_NOISE) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return f + sigma * rng.standard_normal(f.shape[0])


def _apply_mask(y: np.ndarray, mask: np.ndarray) -> np.ndarray:
    y = y.copy()
    y[mask == 0] = np.nan
    return y


def merged_grid(t_train: np.ndarray, t_test: np.ndarray):
    """Sorted union of training and test times; test points become missing
    observations (supplement PAPER.md:255). Ties keep both points (reading Z12)."""
    t = np.concatenate([t_train, t_test])
    m = np.concatenate([np.ones(t_train.shape[0], np.uint8), np.zeros(t_test.shape[0], np.uint8)])
    order = np.argsort(t, kind="stable")
    return t[order], m[order], order


def config1(n_train: int = 1000, n_test: int = 200) -> Workload:
    """C1: Matern-3/2, 1000 train + 200 test points equally spaced on (0, 4)."""
    t_tr = 4.0 * np.arange(1, n_train + 1) / (n_train + 1)
    t_te = 4.0 * np.arange(1, n_test + 1) / (n_test + 1)
    t, mask, _ = merged_grid(t_tr, t_te)
    y = _apply_mask(_noisy(sinusoid(t), 0.1), mask)
    return Workload("C1", [Component("matern32", 1.0, 0.5)], 0.01, t, y, mask)


def jittered_grid(n: int, h: float = H_FINE, jitter: float = 0.45, seed: int = SEED_JITTER) -> np.ndarray:
    """t_i = (i + 1/2 + u_i) h, u_i ~ U(-jitter, jitter): irregular but sorted."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.uniform(-jitter, jitter, n)
    return (np.arange(n, dtype=np.float64) + 0.5 + u) * h


def config2(n_train: int = 2 ** 20, n_test: int = 10_000) -> Workload:
    """C2: Matern-5/2, 2^20 jittered training times + 10,000 equally spaced test times."""
    t_tr = jittered_grid(n_train)
    T = n_train * H_FINE
    t_te = T * np.arange(1, n_test + 1) / (n_test + 1)
    t, mask, _ = merged_grid(t_tr, t_te)
    y = _apply_mask(_noisy(sinusoid(t), 0.1), mask)
    return Workload("C2", [Component("matern52", 1.0, 0.5)], 0.01, t, y, mask)


def bernoulli_mask(n: int, p_missing: float = 1.0 / 16, seed: int = SEED_MASK) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.random(n) >= p_missing).astype(np.uint8)


def metric_workload(n: int = 2 ** 24, uniform: bool = False, kind: str = "matern52") -> Workload:
    """Headline metric (BASELINE.json): Matern-5/2 at N = 2^24, jittered times
    at the paper's finest density (T = N h), 1/16 Bernoulli-missing points."""
    if uniform:
        t = np.arange(n, dtype=np.float64) * H_FINE
    else:
        t = jittered_grid(n)
    mask = bernoulli_mask(n)
    y = _apply_mask(_noisy(sinusoid(t), 0.1), mask)
    return Workload(f"metric_{kind}_{'uniform' if uniform else 'irregular'}_N{n}",
                    [Component(kind, 1.0, 0.5)], 0.01, t, y, mask,
                    uniform_dt=H_FINE if uniform else 0.0)


def config3(n: int = 2 ** 22, order: int = 6, irregular: bool = False) -> Workload:
    """C3: RBF Taylor order 6, uniform dt = h, every 16th point missing.
    irregular=True: the jittered grid of the metric workload instead (device Pade path)."""
    t = jittered_grid(n) if irregular else np.arange(n, dtype=np.float64) * H_FINE
    mask = (np.arange(n) % 16 != 15).astype(np.uint8)
    y = _apply_mask(_noisy(sinusoid(t), 0.1), mask)
    return Workload("C3" + ("_irregular" if irregular else ""), [Component("rbf", 1.0, 0.5, order=order)], 0.01,
                    t, y, mask, uniform_dt=0.0 if irregular else H_FINE)


def co2_like(t: np.ndarray) -> np.ndarray:
    """Smooth multi-scale series with a yearly period (time unit = year)."""
    return (2 * np.sin(2 * np.pi * t / 50) + 1.5 * np.sin(2 * np.pi * t / 13 + 0.3)
            + 3 * np.sin(2 * np.pi * t) + 0.8 * np.sin(4 * np.pi * t + 1) + 0.3 * np.cos(6 * np.pi * t))


def config4(n: int = 2 ** 24, harmonics: int = 6, irregular: bool = False) -> Workload:
    """C4: Periodic(J=6) + Matern-3/2 trend, weekly cadence.  The
    time unit is the WEEK so the grid t_k = k is exactly uniform (dt = 1): period
    52 weeks, trend lengthscale 20 years = 1040 weeks."""
    t = jittered_grid(n, h=1.0) if irregular else np.arange(n, dtype=np.float64)
    mask = (np.arange(n) % 16 != 15).astype(np.uint8)
    y = _noisy(co2_like(t / 52.0), 0.3)
    y = (y - y.mean()) / y.std()
    y = _apply_mask(y, mask)
    comps = [Component("periodic", 4.0, 1.0, period=52.0, order=harmonics),
             Component("matern32", 10.0, 20.0 * 52.0)]
    return Workload("C4" + ("_irregular" if irregular else ""), comps, 0.09, t, y, mask,
                    uniform_dt=0.0 if irregular else 1.0)


def co2_product(n: int = 3192, order: int = 2) -> Workload:
    """The paper's CO2 model C_Per x C_Mat + C_Mat: quasi-periodic
    (J harmonics x Matern-3/2) + Matern-3/2 trend, d = 4 (J + 1) + 2 = 10 / 14 / 18 for
    J = 1 / 2 / 3; weekly grid in weeks (exact uniform dt = 1), 1/16 missing."""
    t = np.arange(n, dtype=np.float64)
    mask = (np.arange(n) % 16 != 15).astype(np.uint8)
    y = _noisy(co2_like(t / 52.0), 0.3)
    y = (y - y.mean()) / y.std()
    y = _apply_mask(y, mask)
    comps = [Component("quasiperiodic", 2.0, 1.0, period=52.0, order=order, mat_lengthscale=300.0, mat_nu2=3),
             Component("matern32", 10.0, 1040.0)]
    return Workload(f"co2_product_J{order}", comps, 0.09, t, y, mask, uniform_dt=1.0)


def random_problem(seed: int, n: int, kind: str = "matern52", p_missing: float = 0.3,
                   ties: int = 0, dt_scale: float = 0.05, lengthscale: Optional[float] = None,
                   variance: Optional[float] = None, noise_var: Optional[float] = None,
                   first_missing: Optional[bool] = None) -> Workload:
    """Small random problem for parity / edge-case tests: exponential gaps,
    optional exact ties (dt = 0), random missing pattern, random hyper-parameters."""
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    gaps = rng.exponential(dt_scale, n)
    gaps[0] = rng.uniform(0, 1)
    if ties > 0 and n > 1:
        idx = rng.choice(np.arange(1, n), size=min(ties, n - 1), replace=False)
        gaps[idx] = 0.0
    t = np.cumsum(gaps)
    mask = (rng.random(n) >= p_missing).astype(np.uint8)
    if first_missing is not None and n > 0:
        mask[0] = 0 if first_missing else 1
    ell = lengthscale if lengthscale is not None else float(rng.uniform(0.2, 2.0))
    var = variance if variance is not None else float(rng.uniform(0.5, 3.0))
    r = noise_var if noise_var is not None else float(rng.uniform(0.01, 0.5))
    f = np.sin(3 * t) + 0.5 * np.cos(7 * t)
    y = f + np.sqrt(r) * rng.standard_normal(n)
    y = _apply_mask(y, mask)
    return Workload(f"rand{seed}_{kind}_N{n}", [Component(kind, var, ell)], r, t, y, mask)
