"""CPU-only tests of the C-ABI library (no GPU): the shared library loads and
exports every symbol include/pssgp.h declares, host-side model construction
matches the oracle's SSM through basis-invariant quantities, and the
discretisation the kernels run (pssgp_debug_discretize calls the same
__host__ __device__ function) matches the oracle's Van Loan on the library's
own model matrices.
"""
import math
import os
import re

import numpy as np
import pytest

import oracle
import synth
from oracle import ssm as ossm

import paper_2102_09964_b200 as P
from paper_2102_09964_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "pssgp.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pssgp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    names = header_functions()
    assert len(names) >= 19
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.SIGNATURES)  # the binding covers the whole ABI


def test_create_errors():
    with pytest.raises(P.PssgpError) as e:
        P.pssgp_create([synth.Component("matern52", 1.0, 0.5)], -1.0)
    assert e.value.status == _native.PSSGP_E_ARG
    with pytest.raises(P.PssgpError) as e:
        P.pssgp_create([synth.Component("matern52", 0.0, 0.5)], 0.1)
    assert e.value.status == _native.PSSGP_E_ARG


def _lib_ssm(h):
    s = P.pssgp_get_ssm(h)
    return ossm.SSM(s["G"], np.zeros((s["G"].shape[0], 1)), 0.0, s["H"], s["Pinf"], Wmat=s["W"]), s


@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
def test_matern_model_reconstructs_kernel(kind):
    comp = synth.Component(kind, 1.7, 0.6)
    m = P.Model([comp], 0.1)
    lm, s = _lib_ssm(m.h)
    taus = np.linspace(0, 3.0, 40)
    np.testing.assert_allclose(ossm.ssm_kernel(lm, taus), ossm.kernel_value(comp, taus), atol=1e-12 * 1.7)
    # stationarity of the library's model: G P + P G^T + W = 0
    res = s["G"] @ s["Pinf"] + s["Pinf"] @ s["G"].T + s["W"]
    assert np.max(np.abs(res)) < 1e-12 * np.max(np.abs(s["W"]))


def test_rbf_and_sum_models():
    comp = synth.Component("rbf", 1.0, 0.5, order=3)
    m = P.Model([comp], 0.1, uniform_dt=synth.H_FINE)
    lm, s = _lib_ssm(m.h)
    om = ossm.build([comp])
    taus = np.linspace(0, 2.0, 30)
    np.testing.assert_allclose(ossm.ssm_kernel(lm, taus), ossm.ssm_kernel(om, taus), rtol=1e-9, atol=1e-12)
    comps = [synth.Component("periodic", 4.0, 1.0, period=1.0, order=6), synth.Component("matern32", 10.0, 20.0)]
    m = P.Model(comps, 0.09, uniform_dt=1 / 52)          # C4: d = 16, warp-per-chain path
    assert m.state_dim == 16
    lm, s = _lib_ssm(m.h)
    om = ossm.build(comps)
    taus = np.linspace(0, 3.0, 31)
    np.testing.assert_allclose(ossm.ssm_kernel(lm, taus), ossm.ssm_kernel(om, taus), rtol=1e-10, atol=1e-12)
    F, Q = m.discretize(1 / 52)
    Fo, Qo = oracle.discretize(lm, 1 / 52)
    assert np.max(np.abs(F - Fo)) < 1e-13 and np.max(np.abs(Q - Qo)) < 1e-13 * np.max(np.abs(Qo))
    with pytest.raises(P.PssgpError):
        m.discretize(0.5 / 52)                            # irregular dt: no device discretisation
    # every d = 4 ... 20 is compiled (north_star "d = 2..~20"); d = 22 is not
    for order in (7, 9, 11):
        assert P.Model([synth.Component("rbf", 1.0, 0.5, order=order)], 0.1, uniform_dt=0.01).state_dim == order
    assert P.Model([synth.Component("periodic", 1.0, 1.0, period=1.0, order=6),
                    synth.Component("matern12", 1.0, 1.0)], 0.1).state_dim == 15
    with pytest.raises(P.PssgpError):
        P.Model([synth.Component("periodic", 1.0, 1.0, period=1.0, order=10)], 0.1, uniform_dt=0.01)


@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
@pytest.mark.parametrize("dt", [0.0, 1e-9, 2.4e-7, 1.22e-4, 1e-3, 0.02, 0.3, 1.0, 2.5, 8.0, 40.0])
def test_closed_form_discretisation_vs_oracle(kind, dt):
    comp = synth.Component(kind, 1.3, 0.5)
    m = P.Model([comp], 0.1)
    lm, s = _lib_ssm(m.h)
    F, Q = m.discretize(dt)
    Fo, Qo = oracle.discretize(lm, dt)
    assert np.max(np.abs(F - Fo)) <= 2e-14 * max(1.0, np.max(np.abs(Fo)))
    qs = np.max(np.abs(s["Pinf"]))
    assert np.max(np.abs(Q - Qo)) <= 1e-14 * qs
    big = np.abs(Qo) > 1e-3 * max(np.max(np.abs(Qo)), 1e-300)
    if big.any():
        assert np.max(np.abs(Q - Qo)[big] / np.abs(Qo)[big]) < 1e-10


def test_uniform_dt_table_vs_oracle():
    for comp, dt in [(synth.Component("matern52", 1.0, 0.5), synth.H_FINE),
                     (synth.Component("rbf", 1.0, 0.5, order=3), synth.H_FINE),
                     (synth.Component("rbf", 1.0, 1.5, order=2), 0.01),
                     (synth.Component("rbf", 1.0, 0.5, order=6), synth.H_FINE),
                     (synth.Component("matern32", 2.0, 0.3), 0.05)]:
        m = P.Model([comp], 0.1, uniform_dt=dt)
        lm, s = _lib_ssm(m.h)
        F, Q = m.discretize(dt)
        Fo, Qo = oracle.discretize(lm, dt)
        assert np.max(np.abs(F - Fo)) <= 1e-13 * max(1.0, np.max(np.abs(Fo)))
        assert np.max(np.abs(Q - Qo)) <= 1e-12 * max(np.max(np.abs(Qo)), 1e-300)


def test_irregular_dt_unsupported_for_non_matern():
    m = P.Model([synth.Component("rbf", 1.0, 0.5, order=2)], 0.1, uniform_dt=0.01)
    with pytest.raises(P.PssgpError) as e:
        m.discretize(0.02)
    assert e.value.status == _native.PSSGP_E_UNSUPPORTED


def test_aggregate_bytes():
    m = P.Model([synth.Component("matern52", 1.0, 0.5)], 0.1)
    assert P.pssgp_aggregate_bytes(m.h, 0) == 27 * 8
    assert P.pssgp_aggregate_bytes(m.h, 1) == (18 + 1) * 8            # smoother aggregate + NLL partial
    m = P.Model([synth.Component("rbf", 1.0, 0.5, order=6)], 0.1, uniform_dt=0.01)
    assert P.pssgp_aggregate_bytes(m.h, 0) == (3 * 36 + 12) * 8     # wide path: full matrices
    assert P.pssgp_aggregate_bytes(m.h, 1) == (2 * 36 + 6 + 1) * 8


def test_quasiperiodic_model_matches_oracle():
    for J in (1, 2, 3):
        w = synth.co2_product(n=10, order=J)
        m = P.Model(w.components, w.noise_var, uniform_dt=1.0)
        assert m.state_dim == 4 * (J + 1) + 2
        lm, s = _lib_ssm(m.h)
        om = ossm.build(w.components)
        taus = np.linspace(0, 200.0, 41)
        np.testing.assert_allclose(ossm.ssm_kernel(lm, taus), ossm.ssm_kernel(om, taus), rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("comps", [
    [synth.Component("rbf", 1.0, 0.5, order=2)],
    [synth.Component("rbf", 1.3, 0.8, order=3)],
    [synth.Component("matern12", 1.0, 0.3), synth.Component("matern32", 2.0, 1.5)],
    [synth.Component("periodic", 1.5, 1.0, period=0.7, order=0)]])
@pytest.mark.parametrize("dt", [0.0, 1e-9, 2.4e-7, 1.22e-4, 1e-3, 0.02, 0.3, 1.0, 2.5, 8.0])
def test_pade_discretisation_vs_oracle(comps, dt):
    """kPade mode (no closed form, uniform_dt = 0): F = expm(G dt) by [7/7] Pade on the scaled
    step and Q by the Taylor series of the Lyapunov ODE, composed by doubling (taylor_fq),
    host-compiled from the same device source, vs the oracle's Pade-13 + sub-stepped Van Loan."""
    m = P.Model(comps, 0.1)
    assert m.state_dim <= 3
    lm, s = _lib_ssm(m.h)
    F, Q = m.discretize(dt)
    Fo, Qo = oracle.discretize(lm, dt)
    assert np.max(np.abs(F - Fo)) <= 1e-13 * max(1.0, np.max(np.abs(Fo)))
    assert np.max(np.abs(Q - Qo)) <= 1e-13 * np.max(np.abs(s["Pinf"]))
    if 0.0 < dt <= 0.02:
        # small steps: every entry of Q to relative accuracy (no cancellation; the stationary
        # shortcut P_inf - F P_inf F^T fails exactly here)
        big = np.abs(Qo) > 1e-280
        if big.any():
            assert np.max(np.abs(Q - Qo)[big] / np.abs(Qo)[big]) <= 1e-10
    if dt == 0.0:
        assert np.array_equal(F, np.eye(m.state_dim)) and np.all(Q == 0.0)


def test_host_side_argument_errors():
    """Argument validation happens on the host, before any device work (no GPU needed)."""
    m = P.Model([synth.Component("matern52", 1.0, 0.5)], 0.1)
    lib = _native.lib()
    one = np.zeros(4)
    ptr = one.ctypes.data
    assert lib.pssgp_nll_grad(m.h, 4, ptr, ptr, ptr, ptr, None, None) == _native.PSSGP_E_ARG     # grad NULL
    assert lib.pssgp_nll_grad(m.h, -1, ptr, ptr, ptr, ptr, ptr, None) == _native.PSSGP_E_ARG     # N < 0
    assert lib.pssgp_predict(m.h, -1, ptr, ptr, 1, ptr, ptr, ptr, ptr, None) == _native.PSSGP_E_ARG
    assert lib.pssgp_predict(m.h, 4, None, ptr, 1, ptr, ptr, ptr, ptr, None) == _native.PSSGP_E_ARG
    assert lib.pssgp_posterior_batched(m.h, 0, ptr, None, None, None, 4, ptr, ptr, ptr, ptr, ptr, ptr,
                                       None) == _native.PSSGP_E_ARG                                # nseg < 1
    r = P.Model([synth.Component("rbf", 1.0, 0.5, order=3)], 0.1)      # no uniform grid declared
    assert lib.pssgp_nll_grad(r.h, 4, ptr, ptr, ptr, ptr, ptr, None) == _native.PSSGP_E_UNSUPPORTED
    assert lib.pssgp_posterior_batched(r.h, 1, ptr, None, None, None, 4, ptr, ptr, ptr, ptr, ptr, ptr,
                                       None) == _native.PSSGP_E_UNSUPPORTED
    assert P.pssgp_last_error(r.h) != ""


def test_num_params_order():
    """pssgp_num_params (include/pssgp.h): 2 per Matern / RBF, 3 per periodic, 4 per quasi-periodic,
    + log noise - the order of oracle.grad.param_names."""
    from oracle import grad as og
    for comps in ([synth.Component("matern52", 1.0, 0.5)],
                  [synth.Component("periodic", 4.0, 1.0, period=1.0, order=6), synth.Component("matern32", 10.0, 20.0)],
                  [synth.Component("quasiperiodic", 2.0, 1.0, period=52.0, order=2, mat_lengthscale=300.0, mat_nu2=3),
                   synth.Component("matern32", 10.0, 1040.0)],
                  [synth.Component("rbf", 1.0, 0.5, order=6)]):
        m = P.Model(comps, 0.1, uniform_dt=0.01)
        assert m.num_params == len(og.param_names(comps))
        # Model.theta (the row layout of the batched per-series calls) = the oracle's theta0
        np.testing.assert_allclose(m.theta, og.theta0(comps, 0.1), rtol=0, atol=1e-15)


def test_no_unenclosed_lane_strided_loops():
    """ptxas may drop a __syncwarp after a lane-strided loop with lane-dependent trip counts without
    re-converging the warp ("A compiler finding"): scan the SASS of every built kernel
    for such loops outside any BSSY/BSYNC region; the only ones allowed are global copies that end
    in EXIT (kw_scan_*) and reductions that continue with re-converging shuffles (k_grad_contract)."""
    import glob
    import shutil
    import subprocess
    import sys
    objs = sorted(glob.glob(os.path.join(os.path.dirname(P.__file__), "build", "*.o")))
    if not objs or shutil.which("cuobjdump") is None:
        pytest.skip("no built objects / cuobjdump")
    tool = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "sass_divergent_loops.py")
    out = subprocess.run([sys.executable, tool, *objs], capture_output=True, text=True, check=True).stdout
    bad = [ln for ln in out.splitlines()
           if " loop " in ln and not ("kw_scan_" in ln and "then: EXIT" in ln) and "k_grad_contract" not in ln]
    assert not bad, "\n".join(bad[:10])
