"""Operator algebra of the paper's parallel formulation (oracle/elements.py),
pinned against mathematics, not against itself:

  * associativity, PAPER.md:326 ("we can select an arbitrary grouping") and
    PAPER.md:431: every Catalan bracketing of n <= 6 random tuples agrees
    (C, J, L symmetric, SURVEY.md finding 3);
  * identities (I, 0, 0, 0, 0) and (I, 0, 0);
  * Prop. 1: the prefix scan of the filter
    elements equals the sequential Kalman filter of the C oracle
    (b*_k = xbar_k, C*_k = P_k), including missing steps;
  * Prop. 2: suffix scan of smoother elements equals RTS;
  * global prefixes collapse to (0, xbar_k, P_k, 0, 0) and global suffixes to
    (0, ms_k, Ps_k) (SURVEY.md finding 2; consequence of A_1 = 0, Eq. (7));
  * tree (Blelloch) scan == sequential scan.
"""
import functools

import numpy as np
import pytest

import oracle
import synth
from oracle import elements as el
from oracle import ssm


def rand_sym(rng, n, psd=True):
    A = rng.standard_normal((n, n))
    return A @ A.T / n if psd else (A + A.T) / 2


def rand_filter_elem(rng, n):
    return (rng.standard_normal((n, n)) * 0.7, rng.standard_normal(n), rand_sym(rng, n),
            rng.standard_normal(n), rand_sym(rng, n))


def rand_smoother_elem(rng, n):
    return (rng.standard_normal((n, n)) * 0.7, rng.standard_normal(n), rand_sym(rng, n))


def all_bracketings(items, op):
    if len(items) == 1:
        return [items[0]]
    out = []
    for s in range(1, len(items)):
        for a in all_bracketings(items[:s], op):
            for b in all_bracketings(items[s:], op):
                out.append(op(a, b))
    return out


def max_dev(results):
    ref = results[0]
    return max(max(np.max(np.abs(x - y)) for x, y in zip(r, ref)) for r in results)


@pytest.mark.parametrize("n", [1, 2, 3, 6])
def test_filter_operator_associative(n):
    rng = np.random.default_rng(n)
    elems = [rand_filter_elem(rng, n) for _ in range(6)]
    res = all_bracketings(elems, el.filter_combine)
    assert len(res) == 42
    scale = max(np.max(np.abs(x)) for x in res[0])
    assert max_dev(res) < 1e-10 * scale


def test_filter_operator_needs_symmetry():
    """SURVEY.md finding 3: with non-symmetric C, J re-bracketing changes the result
    by O(1) — documents why symmetry is kept structurally (packed storage)."""
    rng = np.random.default_rng(7)
    n = 3
    elems = [(rng.standard_normal((n, n)), rng.standard_normal(n), rng.standard_normal((n, n)),
              rng.standard_normal(n), rng.standard_normal((n, n))) for _ in range(4)]
    res = all_bracketings(elems, el.filter_combine)
    assert max_dev(res) > 1e-3


@pytest.mark.parametrize("n", [1, 3, 6])
def test_smoother_operator_associative(n):
    rng = np.random.default_rng(10 + n)
    elems = [rand_smoother_elem(rng, n) for _ in range(6)]
    res = all_bracketings(elems, el.smoother_combine)
    scale = max(np.max(np.abs(x)) for x in res[0])
    assert max_dev(res) < 1e-12 * scale


def test_identities():
    rng = np.random.default_rng(1)
    for n in (1, 3):
        e = rand_filter_elem(rng, n)
        I = el.filter_identity(n)
        for a, b in zip(el.filter_combine(I, e), e):
            np.testing.assert_allclose(a, b, atol=1e-14)
        for a, b in zip(el.filter_combine(e, I), e):
            np.testing.assert_allclose(a, b, atol=1e-14)
        s = rand_smoother_elem(rng, n)
        Is = el.smoother_identity(n)
        for a, b in zip(el.smoother_combine(Is, s), s):
            np.testing.assert_allclose(a, b, atol=1e-15)
        for a, b in zip(el.smoother_combine(s, Is), s):
            np.testing.assert_allclose(a, b, atol=1e-15)


def test_spec_hand_elements():
    """SPEC.md:312 observed element and SPEC.md:341 smoother element (scalar)."""
    F = [None, np.array([[1.0]])]
    Q = [None, np.array([[1.0]])]
    e = el.filter_elements(F, Q, np.array([1.0]), np.array([[1.0]]), 1.0, np.array([0.0, 2.0]),
                           np.array([0, 1], np.uint8))[1]
    A, b, C, eta, J = (float(np.ravel(x)[0]) for x in e)
    assert (A, b, C, eta, J) == (0.5, 1.0, 0.5, 1.0, 0.5)
    xf = np.array([[3.0], [0.0]]); Pf = np.array([[[1.0]], [[1.0]]])
    E, g, L = el.smoother_elements(F, Q, xf, Pf)[0]
    assert float(E[0, 0]) == 0.5 and float(g[0]) == 1.5 and float(L[0, 0]) == 0.5


def _discretized(w, m):
    F = [None]; Q = [None]
    for k in range(1, w.N):
        Fk, Qk = oracle.discretize(m, w.t[k] - w.t[k - 1])
        F.append(Fk); Q.append(Qk)
    return F, Q


@pytest.mark.parametrize("kind,p_missing,first_missing", [("matern32", 0.3, True), ("matern52", 0.3, False),
                                                          ("matern52", 1.0, None), ("matern12", 0.0, None)])
def test_prop1_prop2_vs_sequential_oracle(kind, p_missing, first_missing):
    w = synth.random_problem(31, 64, kind=kind, p_missing=p_missing, ties=2, first_missing=first_missing)
    m = ssm.build(w.components)
    o = oracle.kf_rts(m, w.noise_var, w.t, w.y, w.mask, moments=True)
    F, Q = _discretized(w, m)
    fe = el.filter_elements(F, Q, m.H, m.Pinf, w.noise_var, w.y, w.mask)
    scale = np.max(np.abs(m.Pinf))
    for scan in (lambda e: el.sequential_scan(e, el.filter_combine),
                 lambda e: el.tree_scan(e, el.filter_combine, el.filter_identity(m.n))):
        pref = scan(fe)
        for k in range(w.N):
            A, b, C, eta, J = pref[k]
            np.testing.assert_allclose(b, o["xf"][k], atol=1e-9 * np.sqrt(scale))
            np.testing.assert_allclose(C, o["Pf"][k], atol=1e-9 * scale)
            # global prefix collapse (A_1 = 0 propagates)
            assert np.max(np.abs(A)) == 0.0 and np.max(np.abs(eta)) == 0.0 and np.max(np.abs(J)) == 0.0
    se = el.smoother_elements(F, Q, o["xf"], o["Pf"])
    for scan in (lambda e: el.sequential_scan(e, el.smoother_combine, reverse=True),
                 lambda e: el.tree_scan(e, el.smoother_combine, el.smoother_identity(m.n), reverse=True)):
        suf = scan(se)
        for k in range(w.N):
            E, g, L = suf[k]
            np.testing.assert_allclose(g, o["xs"][k], atol=1e-9 * np.sqrt(scale))
            np.testing.assert_allclose(L, o["Ps"][k], atol=1e-9 * scale)
            assert np.max(np.abs(E)) == 0.0


def test_tree_scan_matches_sequential_on_addition():
    xs = list(np.arange(1.0, 14.0))
    np.testing.assert_array_equal(el.tree_scan(xs, lambda a, b: a + b, 0.0), np.cumsum(xs))
    np.testing.assert_array_equal(el.tree_scan(xs, lambda a, b: a + b, 0.0, reverse=True), np.cumsum(xs[::-1])[::-1])
    s = el.tree_scan([np.array([2.0, 1.0])], lambda a, b: a * b, np.array([1.0, 1.0]))  # N = 1
    np.testing.assert_array_equal(s[0], [2.0, 1.0])
