"""Regenerate tests/golden/rbf_taylor_pins.json: the RBF Taylor state-space construction of
reading Z7 evaluated in 50-digit arithmetic with mpmath, written
from the definition and independent of oracle/ssm.py (which uses numpy.roots in fp64):

  1/S(w) with S(w) = s2 sqrt(2 pi) ell exp(-ell^2 w^2 / 2), Taylor-expanded to order n in
  ell^2 w^2 / 2, is with s = i w the polynomial p(s) = sum_j (ell^2/2)^j (-s^2)^j / j!;
  a(s) = the monic polynomial of the n left-half-plane roots of p, so that
  p(s) = c a(s) a(-s) with c = (ell^2/2)^n / n!, and S(w) ~ q / |a(i w)|^2 with
  q = s2 sqrt(2 pi) ell n! (2 / ell^2)^n.

usage: python tools/gen_rbf_pins.py     (rewrites the golden file)
"""
import json
import os

import mpmath as mp

mp.mp.dps = 50
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "rbf_taylor_pins.json")


def spectral_factor(n, ell, s2=1):
    ell = mp.mpf(ell)
    # p(s) coefficients, highest degree first (degree 2n, only even powers)
    coeffs = [mp.mpf(0)] * (2 * n + 1)
    for j in range(n + 1):
        coeffs[2 * n - 2 * j] = (ell ** 2 / 2) ** j * (-1) ** j / mp.factorial(j)
    roots = mp.polyroots(coeffs, maxsteps=500, extraprec=400)
    left = sorted([r for r in roots if mp.re(r) < 0], key=lambda r: (mp.re(r), mp.im(r)))
    assert len(left) == n
    a = [mp.mpc(1)]
    for r in left:                         # multiply by (s - r)
        a = [x - r * y for x, y in zip(a + [0], [0] + a)]
    a = [mp.re(x) for x in a]              # conjugate pairs: real coefficients
    q = s2 * mp.sqrt(2 * mp.pi) * ell * mp.factorial(n) * (2 / ell ** 2) ** n
    return a, q


def main():
    cases = []
    for n, ell in [(4, 1.0), (6, 1.0), (6, 0.5), (8, 1.0)]:
        a, q = spectral_factor(n, ell)
        cases.append({"order": n, "lengthscale": ell, "variance": 1.0,
                      "a_monic_high_to_low": [mp.nstr(x, 30) for x in a], "q": mp.nstr(q, 30)})
    json.dump({"source": "tools/gen_rbf_pins.py (mpmath, 50 digits); construction of DESIGN.md reading Z7",
               "cases": cases}, open(OUT, "w"), indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
