"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element, on seeded synthetic inputs.  Tolerances (north_star, BASELINE.json;
measures = SURVEY.md §8(c) reading Z14):
    mean: normwise   max|dm| / max|m_ref|      <= 1e-8
    var : elementwise max|dv / v_ref|           <= 1e-8
    nll : |dNLL| / |NLL_ref|                   <= 1e-9
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2102_09964_b200 as P
from paper_2102_09964_b200 import _native

pytestmark = pytest.mark.gpu

MEAN_TOL, VAR_TOL, NLL_TOL = 1e-8, 1e-8, 1e-9


def to_dev(w, dev="cuda:0"):
    return (torch.from_numpy(w.t).to(dev), torch.from_numpy(w.y).to(dev), torch.from_numpy(w.mask).to(dev))


def run_gpu(w, **kw):
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt, **kw)
    t, y, mk = to_dev(w)
    mean, var, nll = m.posterior(t, y, mk)
    m.check()
    return mean.cpu().numpy(), var.cpu().numpy(), float(nll.cpu()[0]), m


def errors(g, o):
    mean, var, nll = g
    em = np.max(np.abs(mean - o["mean"])) / max(np.max(np.abs(o["mean"])), 1e-300)
    ev = np.max(np.abs(var - o["var"]) / np.abs(o["var"]))
    scale = abs(o["nll"]) if abs(o["nll"]) > 1e-12 else 1.0
    en = abs(nll - o["nll"]) / scale
    return em, ev, en


def assert_parity(w, o=None, **kw):
    if o is None:
        o = oracle.posterior(w)
    mean, var, nll, m = run_gpu(w, **kw)
    if w.mask.sum() == 0:
        assert np.max(np.abs(mean)) == 0.0 and nll == 0.0
        np.testing.assert_allclose(var, o["var"], rtol=VAR_TOL)
        return m
    em, ev, en = errors((mean, var, nll), o)
    assert em <= MEAN_TOL and ev <= VAR_TOL and en <= NLL_TOL, (em, ev, en)
    return m


def test_config1_full(cuda_device):
    assert_parity(synth.config1())


@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52"])
@pytest.mark.parametrize("N", [1, 2, 3, 31, 33, 257, 1000, 4099, 30011])
def test_random_sizes(cuda_device, kind, N):
    w = synth.random_problem(N % 97, N, kind=kind, p_missing=0.3, ties=min(3, N // 10))
    assert_parity(w)


@pytest.mark.parametrize("chain_len", [1, 2, 5, 16, 17])
def test_small_chains_many_blocks(cuda_device, chain_len):
    """Tiny chains -> hundreds of CTAs and multi-pass single-CTA carry scans."""
    w = synth.random_problem(5, 70001, kind="matern52", p_missing=0.2, ties=4, dt_scale=0.01)
    assert_parity(w, chain_len=chain_len)


@pytest.mark.parametrize("p_missing,first_missing", [(0.0, None), (1.0, None), (0.5, True), (0.5, False), (0.97, True)])
def test_missing_patterns(cuda_device, p_missing, first_missing):
    w = synth.random_problem(8, 3001, kind="matern32", p_missing=p_missing, first_missing=first_missing)
    assert_parity(w)


def test_uniform_fast_path(cuda_device):
    w = synth.metric_workload(2 ** 16, uniform=True)
    assert_parity(w)


def test_large_gaps_and_far_field(cuda_device):
    """Large gaps (dt >> lengthscale) and isolated observations: prior reversion."""
    w = synth.random_problem(12, 5000, kind="matern52", p_missing=0.6, dt_scale=0.8, lengthscale=0.3)
    assert_parity(w)


def test_config2_full(cuda_device):
    w = synth.config2()
    assert_parity(w)


@pytest.mark.slow
def test_metric_full_size(cuda_device):
    """Headline configuration (N = 2^24, bench.py's launch configuration)."""
    w = synth.metric_workload(2 ** 24)
    assert_parity(w)


def test_nll_only_matches_posterior(cuda_device):
    w = synth.random_problem(2, 20000, kind="matern52", p_missing=0.1)
    m = P.Model(w.components, w.noise_var)
    t, y, mk = to_dev(w)
    _, _, nll_a = m.posterior(t, y, mk)
    nll_b = m.nll(t, y, mk)
    m.check()
    assert float(nll_a.cpu()[0]) == float(nll_b.cpu()[0])


def test_deterministic(cuda_device):
    w = synth.random_problem(3, 100000, kind="matern52", p_missing=0.1)
    m = P.Model(w.components, w.noise_var)
    t, y, mk = to_dev(w)
    a = [x.clone() for x in m.posterior(t, y, mk)]
    b = m.posterior(t, y, mk)
    for u, v in zip(a, b):
        assert torch.equal(u, v)


def test_host_api_matches_device(cuda_device):
    w = synth.random_problem(4, 50000, kind="matern32", p_missing=0.2)
    m = P.Model(w.components, w.noise_var)
    t, y, mk = to_dev(w)
    mean, var, nll = m.posterior(t, y, mk)
    hm, hv, hn = m.posterior_host(w.t, w.y, w.mask)
    np.testing.assert_array_equal(hm, mean.cpu().numpy())
    np.testing.assert_array_equal(hv, var.cpu().numpy())
    assert hn[0] == float(nll.cpu()[0])


def test_input_errors(cuda_device):
    w = synth.random_problem(6, 5000, kind="matern52", p_missing=0.2)
    m = P.Model(w.components, w.noise_var)
    t = w.t.copy(); t[3001] = t[3000] - 1e-6
    tt, y, mk = to_dev(w)
    tt = torch.from_numpy(t).cuda()
    m.posterior(tt, y, mk)
    with pytest.raises(P.PssgpError) as e:
        m.check()
    assert e.value.status == _native.PSSGP_E_INPUT and e.value.index == 3001
    yb = w.y.copy(); obs = np.nonzero(w.mask)[0]; yb[obs[100]] = np.nan
    m.posterior(to_dev(w)[0], torch.from_numpy(yb).cuda(), mk)
    with pytest.raises(P.PssgpError) as e:
        m.check()
    assert e.value.status == _native.PSSGP_E_INPUT and e.value.index == obs[100]
    m.posterior(*to_dev(w))
    m.check()                                             # error latch was cleared


def test_unsupported_irregular_dt(cuda_device):
    w = synth.random_problem(6, 500, kind="matern52")
    m = P.Model([synth.Component("rbf", 1.0, 0.5, order=3)], 0.1, uniform_dt=0.01)
    m.posterior(*to_dev(w))
    with pytest.raises(P.PssgpError) as e:
        m.check()
    assert e.value.status == _native.PSSGP_E_UNSUPPORTED


@pytest.mark.parametrize("world", [2, 3, 8])
def test_virtual_sharding(cuda_device, world):
    """Time-sharded 3-phase protocol run shard by shard on one GPU (no kernel waits
    on another), exchanging aggregates through device memory; must match the
    unsharded path."""
    w = synth.random_problem(9, 40003, kind="matern52", p_missing=0.2, ties=3)
    ref_mean, ref_var, ref_nll, _ = run_gpu(w)
    from paper_2102_09964_b200 import sharded
    mean, var, nll = sharded.run_virtual(w.components, w.noise_var, w.t, w.y, w.mask, world)
    em = np.max(np.abs(mean - ref_mean)) / np.max(np.abs(ref_mean))
    ev = np.max(np.abs(var - ref_var) / ref_var)
    assert em < 1e-11 and ev < 1e-11
    assert abs(nll - ref_nll) < 1e-11 * abs(ref_nll)
    o = oracle.posterior(w)
    em, ev, en = errors((mean, var, nll), o)
    assert em <= MEAN_TOL and ev <= VAR_TOL and en <= NLL_TOL


def test_misaligned_mask_pointer(cuda_device):
    """A mask view starting at an odd byte address takes the register-prefetch path."""
    w = synth.random_problem(14, 9001, kind="matern52", p_missing=0.3)
    o = oracle.posterior(w)
    m = P.Model(w.components, w.noise_var)
    t, y, _ = to_dev(w)
    big = torch.zeros(w.N + 1, dtype=torch.uint8, device="cuda:0")
    big[1:] = torch.from_numpy(w.mask).cuda()
    mk = big[1:]
    assert mk.data_ptr() % 4 != 0
    mean, var, nll = m.posterior(t, y, mk)
    m.check()
    em, ev, en = errors((mean.cpu().numpy(), var.cpu().numpy(), float(nll.cpu()[0])), o)
    assert em <= MEAN_TOL and ev <= VAR_TOL and en <= NLL_TOL


# ------------------------------------------------------------------ warp-per-chain path (d >= 4, uniform dt)
def _uniform(components, noise_var, n, dt, p_missing=1 / 16, seed=0, f=None):
    t = np.arange(n, dtype=np.float64) * dt
    rng = np.random.default_rng(seed)
    mask = (rng.random(n) >= p_missing).astype(np.uint8)
    base = synth.sinusoid(t) if f is None else f(t)
    y = base + np.sqrt(noise_var) * rng.standard_normal(n)
    y[mask == 0] = np.nan
    return synth.Workload("uniform", components, noise_var, t, y, mask, uniform_dt=dt)


@pytest.mark.parametrize("n", [1, 7, 300, 4097])
def test_wide_rbf6(cuda_device, n):
    """C3-shaped: RBF Taylor order 6 (d = 6), uniform dt = h, 1/16 missing."""
    w = _uniform([synth.Component("rbf", 1.0, 0.5, order=6)], 0.01, n, synth.H_FINE * 64)
    assert_parity(w)


def test_wide_config3_shape(cuda_device):
    w = synth.config3(n=2 ** 15)
    assert_parity(w)


@pytest.mark.parametrize("n", [5, 2000])
def test_wide_config4_shape(cuda_device, n):
    """C4-shaped: periodic J = 6 (d = 14) + Matern-3/2 trend (d = 2) = d 16, weekly cadence."""
    w = synth.config4(n=n)
    assert_parity(w)


@pytest.mark.parametrize("comps,dt", [
    ([synth.Component("matern32", 1.0, 0.7), synth.Component("matern32", 0.5, 3.0)], 0.01),   # d = 4
    ([synth.Component("matern32", 1.0, 0.7), synth.Component("matern52", 0.5, 3.0)], 0.02),   # d = 5
    ([synth.Component("periodic", 1.0, 1.0, period=0.5, order=3), synth.Component("matern32", 1.0, 2.0)], 0.01),  # d = 10
])
def test_wide_sums(cuda_device, comps, dt):
    w = _uniform(comps, 0.05, 3001, dt, p_missing=0.3, seed=3)
    assert_parity(w)


# every compiled state dimension of the warp-per-chain path (pssgp_dims.h: d = 4 ... 20; north_star
# "d = 2..~20"): the odd ones added in round 2 on uniform and jittered grids
_ODD_D = {
    7: [synth.Component("rbf", 1.0, 0.6, order=7)],
    9: [synth.Component("periodic", 1.0, 1.0, period=0.5, order=3), synth.Component("matern12", 0.5, 2.0)],
    11: [synth.Component("periodic", 1.0, 1.0, period=0.5, order=4), synth.Component("matern12", 0.5, 2.0)],
    13: [synth.Component("periodic", 1.0, 1.0, period=0.5, order=5), synth.Component("matern12", 0.5, 2.0)],
    15: [synth.Component("periodic", 1.0, 1.0, period=0.5, order=6), synth.Component("matern12", 0.5, 2.0)],
    17: [synth.Component("periodic", 1.0, 1.0, period=0.5, order=7), synth.Component("matern12", 0.5, 2.0)],
    19: [synth.Component("periodic", 1.0, 1.0, period=0.5, order=8), synth.Component("matern12", 0.5, 2.0)],
}


@pytest.mark.parametrize("d", sorted(_ODD_D))
def test_wide_odd_state_dims(cuda_device, d):
    w = _uniform(_ODD_D[d], 0.05, 2501, 0.01, p_missing=0.25, seed=d)
    m = assert_parity(w)
    assert m.state_dim == d
    wi = _irregular(_ODD_D[d], 0.05, 1201, seed=d)
    assert_parity(wi)


def test_wide_ties_and_small_chains(cuda_device):
    w = _uniform([synth.Component("rbf", 1.0, 0.8, order=4)], 0.02, 5003, 0.01, p_missing=0.25, seed=5)
    w.t[100:103] = w.t[100]           # exact ties (dt = 0)
    w.t[103:] = w.t[103:] - 3 * 0.01  # keep the remaining steps uniform
    w.uniform_dt = 0.01
    assert_parity(w, chain_len=3)


@pytest.mark.parametrize("model", ["rbf6", "per4+m32", "quasi3+m32"])
@pytest.mark.parametrize("world", [2, 3])
def test_wide_virtual_sharding(cuda_device, world, model):
    """Shard phases of the wide path (d = 6 quarters; d = 12 half chains and d = 18 warp chains,
    whose unsharded RTS rescan runs in adjoint form while the shard phase, which has no y, keeps the
    RTS step) against the unsharded posterior."""
    comps = {"rbf6": [synth.Component("rbf", 1.0, 0.5, order=6)],
             "per4+m32": [synth.Component("periodic", 1.5, 1.0, period=0.7, order=4),
                          synth.Component("matern32", 1.0, 2.0)],
             "quasi3+m32": [synth.Component("quasiperiodic", 2.0, 1.0, period=0.5, order=3, mat_lengthscale=3.0,
                                            mat_nu2=3),
                            synth.Component("matern32", 1.0, 2.0)]}[model]
    w = _uniform(comps, 0.01, 6001, 0.002, p_missing=0.2, seed=9)
    ref_mean, ref_var, ref_nll, _ = run_gpu(w)
    from paper_2102_09964_b200 import sharded
    mean, var, nll = sharded.run_virtual(w.components, w.noise_var, w.t, w.y, w.mask, world, uniform_dt=w.uniform_dt)
    assert np.max(np.abs(mean - ref_mean)) / np.max(np.abs(ref_mean)) < 1e-10
    assert np.max(np.abs(var - ref_var) / ref_var) < 1e-10
    assert abs(nll - ref_nll) < 1e-10 * abs(ref_nll)


@pytest.mark.parametrize("order", [1, 2, 3])
def test_co2_product_model(cuda_device, order):
    """NEXT row f3: the paper's CO2 model C_Per x C_Mat + C_Mat, n_x = 10/14/18,
    N = 3192 weekly points (the dataset size of PAPER.md:224)."""
    w = synth.co2_product(n=3192, order=order)
    assert_parity(w)


def test_merge_grid_and_predict(cuda_device):
    """NEXT row f4: device merge equals the stable sorted union (training
    first on ties), and pssgp_predict equals the oracle on the merged grid."""
    rng = np.random.default_rng(21)
    t_tr = np.sort(rng.uniform(0, 4, 5000))
    t_te = np.sort(np.concatenate([rng.uniform(-0.5, 4.5, 1500), t_tr[::97]]))   # includes exact ties
    y_tr = synth.sinusoid(t_tr) + 0.1 * rng.standard_normal(t_tr.shape[0])
    comps = [synth.Component("matern52", 1.0, 0.5)]
    m = P.Model(comps, 0.01)
    dev = "cuda:0"
    T, Y, TE = (torch.from_numpy(a).to(dev) for a in (t_tr, y_tr, t_te))
    n = t_tr.shape[0] + t_te.shape[0]
    tg = torch.empty(n, dtype=torch.float64, device=dev); yg = torch.empty_like(tg)
    mk = torch.empty(n, dtype=torch.uint8, device=dev); idx = torch.empty(t_te.shape[0], dtype=torch.int64, device=dev)
    P.pssgp_merge_grid(m.h, t_tr.shape[0], T, Y, t_te.shape[0], TE, tg, yg, mk, idx)
    m.check()
    t_ref, m_ref, order = synth.merged_grid(t_tr, t_te)
    np.testing.assert_array_equal(tg.cpu().numpy(), t_ref)
    np.testing.assert_array_equal(mk.cpu().numpy(), m_ref)
    pos = np.empty(n, np.int64); pos[order] = np.arange(n)
    np.testing.assert_array_equal(idx.cpu().numpy(), pos[t_tr.shape[0]:])
    mt, vt, nll = m.predict(T, Y, TE)
    m.check()
    y_ref = np.concatenate([y_tr, np.full(t_te.shape[0], np.nan)])[order]
    o = oracle.posterior(synth.Workload("merged", comps, 0.01, t_ref, y_ref, m_ref))
    om, ov = o["mean"][pos[t_tr.shape[0]:]], o["var"][pos[t_tr.shape[0]:]]
    assert np.max(np.abs(mt.cpu().numpy() - om)) / np.max(np.abs(om)) < MEAN_TOL
    assert np.max(np.abs(vt.cpu().numpy() - ov) / ov) < VAR_TOL
    assert abs(float(nll.cpu()[0]) - o["nll"]) < NLL_TOL * abs(o["nll"])
    tb = T.clone(); tb[10] = tb[9] - 1.0                                 # unsorted training times
    P.pssgp_merge_grid(m.h, t_tr.shape[0], tb, Y, t_te.shape[0], TE, tg, yg, mk, idx)
    with pytest.raises(P.PssgpError) as e:
        m.check()
    assert e.value.status == _native.PSSGP_E_INPUT and e.value.index == 10


@pytest.mark.parametrize("kind", ["matern32", "matern52"])
def test_batched_series(cuda_device, kind):
    """NEXT row f2: independent series with their own hyper-parameters in one launch
    (incl. empty and 1-point series, series spanning many chains); each equals the
    oracle on that series alone, NLL per series."""
    rng = np.random.default_rng(31)
    lens = [0, 1, 2, 37, 3200, 0, 5000, 777, 1, 12000, 300]
    ws = []
    for b, n in enumerate(lens):
        ws.append(synth.random_problem(100 + b, n, kind=kind, p_missing=0.2, ties=min(2, n // 10),
                                       lengthscale=float(rng.uniform(0.2, 2.0)), variance=float(rng.uniform(0.5, 3.0)),
                                       noise_var=float(rng.uniform(0.01, 0.3))) if n > 0 else None)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cat = lambda f, dt: np.concatenate([f(w) if w is not None else np.zeros(0, dt) for w in ws])  # noqa: E731
    t = cat(lambda w: w.t, np.float64); y = cat(lambda w: w.y, np.float64); mk = cat(lambda w: w.mask, np.uint8)
    var_b = np.array([w.components[0].variance if w else 1.0 for w in ws])
    ell_b = np.array([w.components[0].lengthscale if w else 1.0 for w in ws])
    r_b = np.array([w.noise_var if w else 0.1 for w in ws])
    m = P.Model([synth.Component(kind, 1.0, 1.0)], 0.1, chain_len=64)
    dev = "cuda:0"
    T, Y, MK = (torch.from_numpy(a).to(dev) for a in (t, y, mk))
    OFF, VB, EB, RB = (torch.from_numpy(a).to(dev) for a in (off, var_b, ell_b, r_b))
    N = t.shape[0]
    mean = torch.empty(N, dtype=torch.float64, device=dev); var = torch.empty_like(mean)
    nll = torch.empty(len(lens), dtype=torch.float64, device=dev)
    P.pssgp_posterior_batched(m.h, len(lens), OFF, VB, EB, RB, N, T, Y, MK, mean, var, nll)
    m.check()
    mean, var, nll = mean.cpu().numpy(), var.cpu().numpy(), nll.cpu().numpy()
    for b, w in enumerate(ws):
        if w is None:
            assert nll[b] == 0.0
            continue
        o = oracle.posterior(w)
        sl = slice(off[b], off[b + 1])
        if w.mask.sum():
            em, ev, en = errors((mean[sl], var[sl], nll[b]), o)
            assert em <= MEAN_TOL and ev <= VAR_TOL and en <= NLL_TOL, (b, em, ev, en)
        else:
            np.testing.assert_allclose(var[sl], o["var"], rtol=VAR_TOL)


def _irregular(comps, noise_var, n, seed, dt_scale=0.02, p_missing=0.3, ties=3):
    base = synth.random_problem(seed, n, kind="matern52", p_missing=p_missing, ties=ties, dt_scale=dt_scale,
                                noise_var=noise_var)
    return synth.Workload(f"irregular_{seed}_{n}", comps, noise_var, base.t, base.y, base.mask)


PADE_MODELS = {
    "rbf3": [synth.Component("rbf", 1.3, 0.8, order=3)],
    "m12+m32": [synth.Component("matern12", 1.0, 0.3), synth.Component("matern32", 2.0, 1.5)],
    "rbf6": [synth.Component("rbf", 1.0, 0.5, order=6)],
    "per3+m32": [synth.Component("periodic", 1.5, 1.0, period=0.7, order=3), synth.Component("matern32", 1.0, 2.0)],
    "per6+m32": [synth.Component("periodic", 4.0, 1.0, period=1.0, order=6), synth.Component("matern32", 10.0, 20.0)],
    "quasi1": [synth.Component("quasiperiodic", 2.0, 1.0, period=0.5, order=1, mat_lengthscale=3.0, mat_nu2=3)],
    # d = 12 in 4 x 4 blocks (the per-block discretisation kw_discretize_blk<12, 4>)
    "quasi2": [synth.Component("quasiperiodic", 2.0, 1.0, period=0.5, order=2, mat_lengthscale=3.0, mat_nu2=3)],
    # d = 14 in blocks of 4, the last one partial (rows 12, 13: the Matern-3/2 trend)
    "quasi2+m32": [synth.Component("quasiperiodic", 2.0, 1.0, period=0.5, order=2, mat_lengthscale=3.0, mat_nu2=3),
                   synth.Component("matern32", 1.0, 2.0)],
}


@pytest.mark.parametrize("name", list(PADE_MODELS))
def test_irregular_pade_models(cuda_device, name):
    """Irregular time grid for models without a closed form (uniform_dt = 0): per-step
    expm by [7/7] Pade scaling and squaring on the device (north_star discretisation
    kernel), thread path for d <= 3 and kw_discretize + warp path above."""
    comps = PADE_MODELS[name]
    n = 20011 if name in ("rbf3", "m12+m32", "rbf6") else 4001
    w = _irregular(comps, 0.05, n, seed=len(name))
    assert_parity(w)


def test_irregular_pade_small_chains_and_sharding(cuda_device):
    w = _irregular(PADE_MODELS["rbf6"], 0.05, 9001, seed=31, dt_scale=0.01)
    assert_parity(w, chain_len=3)
    ref_mean, ref_var, ref_nll, _ = run_gpu(w)
    from paper_2102_09964_b200 import sharded
    for world in (2, 3):
        mean, var, nll = sharded.run_virtual(w.components, w.noise_var, w.t, w.y, w.mask, world)
        assert np.max(np.abs(mean - ref_mean)) / np.max(np.abs(ref_mean)) < 1e-10
        assert np.max(np.abs(var - ref_var) / ref_var) < 1e-10
        assert abs(nll - ref_nll) < 1e-10 * abs(ref_nll)
    w3 = _irregular(PADE_MODELS["rbf3"], 0.05, 9001, seed=32, dt_scale=0.01)
    ref_mean, ref_var, ref_nll, _ = run_gpu(w3)
    mean, var, nll = sharded.run_virtual(w3.components, w3.noise_var, w3.t, w3.y, w3.mask, 3)
    assert np.max(np.abs(mean - ref_mean)) / np.max(np.abs(ref_mean)) < 1e-10
    assert abs(nll - ref_nll) < 1e-10 * abs(ref_nll)


@pytest.mark.parametrize("name,dt_scale", [("rbf3", 1.2e-4), ("m12+m32", 1.2e-4), ("rbf6", 1.2e-4),
                                           ("per3+m32", 1.2e-4), ("rbf3", 2e-6), ("m12+m32", 2e-6),
                                           ("rbf6", 2e-6)])
def test_irregular_pade_fine_grids(cuda_device, name, dt_scale):
    """Fine irregular grids (the paper's finest density h = 1.22e-4 and far below): Q_k is tiny
    next to P_inf, where the stationary shortcut P_inf - F P_inf F^T cancels.
    (per3+m32 at dt ~ 2e-6 spans 6 % of one period: the problem itself is ill-conditioned there,
    the oracle and the dense GP differ by 3e-3 in var, so it is not a parity case.)"""
    comps = PADE_MODELS[name]
    w = _irregular(comps, 0.01, 20011, seed=7, dt_scale=dt_scale)
    assert_parity(w)


def test_handle_reuse_across_entry_points(cuda_device):
    """One handle through predict / batched / posterior with growing sizes (each grows its own
    handle-owned buffer) gives the same results as fresh handles, and destroys cleanly."""
    rng = np.random.default_rng(3)
    comps = [synth.Component("matern52", 1.0, 0.5)]
    m = P.Model(comps, 0.01)
    for n_tr, n_te in [(500, 50), (3000, 700)]:
        t_tr = np.sort(rng.uniform(0, 4, n_tr)); y_tr = synth.sinusoid(t_tr) + 0.1 * rng.standard_normal(n_tr)
        t_te = np.sort(rng.uniform(0, 4, n_te))
        d = lambda a: torch.from_numpy(a).cuda()
        mt, vt, nll = m.predict(d(t_tr), d(y_tr), d(t_te))
        fresh = P.Model(comps, 0.01)
        mt2, vt2, nll2 = fresh.predict(d(t_tr), d(y_tr), d(t_te))
        assert torch.equal(mt, mt2) and torch.equal(vt, vt2) and torch.equal(nll, nll2)
        B = 3
        off = torch.tensor([0, n_tr // 3, 2 * n_tr // 3, n_tr], dtype=torch.int64, device="cuda:0")
        mask = torch.ones(n_tr, dtype=torch.uint8, device="cuda:0")
        mean = torch.empty(n_tr, dtype=torch.float64, device="cuda:0"); var = torch.empty_like(mean)
        nllb = torch.empty(B, dtype=torch.float64, device="cuda:0")
        P.pssgp_posterior_batched(m.h, B, off, None, None, None, n_tr, d(t_tr), d(y_tr), mask, mean, var, nllb)
        m.check()
        w = synth.Workload("reuse", comps, 0.01, t_tr, y_tr, np.ones(n_tr, np.uint8))
        g = m.posterior(d(w.t), d(w.y), d(w.mask))
        m.check()
        o = oracle.posterior(w)
        em, ev, en = errors((g[0].cpu().numpy(), g[1].cpu().numpy(), float(g[2].cpu()[0])), o)
        assert em <= MEAN_TOL and ev <= VAR_TOL and en <= NLL_TOL
        fresh.close()
    m.close()


def test_batched_invalid_offsets(cuda_device):
    """Offsets that do not partition [0, N) are reported (PSSGP_E_INPUT) instead of hanging."""
    m = P.Model([synth.Component("matern32", 1.0, 0.5)], 0.01)
    n = 1000
    t = torch.linspace(0, 1, n, dtype=torch.float64, device="cuda:0")
    y = torch.zeros(n, dtype=torch.float64, device="cuda:0")
    mk = torch.ones(n, dtype=torch.uint8, device="cuda:0")
    mean = torch.empty_like(t); var = torch.empty_like(t)
    nll = torch.empty(2, dtype=torch.float64, device="cuda:0")
    for bad in ([0, 600, 900], [0, 700, 300], [5, 500, n]):
        off = torch.tensor(bad, dtype=torch.int64, device="cuda:0")
        P.pssgp_posterior_batched(m.h, 2, off, None, None, None, n, t, y, mk, mean, var, nll)
        with pytest.raises(P.PssgpError) as e:
            m.check()
        assert e.value.status == _native.PSSGP_E_INPUT


def _mp_van_loan(G, W, dt, dps=40):
    """F, Q at 40 digits (mpmath expm of the Van Loan block matrix) — an independent
    high-precision reference (the fp64 oracle's expm itself carries ~1e-11 error for the
    non-normal balanced RBF-6 drift at dt ~ 0.3)."""
    import mpmath as mp
    mp.mp.dps = dps
    d = G.shape[0]
    C = mp.zeros(2 * d, 2 * d)
    for i in range(d):
        for j in range(d):
            C[i, j] = mp.mpf(G[i, j]) * dt
            C[i, d + j] = mp.mpf(W[i, j]) * dt
            C[d + i, d + j] = -mp.mpf(G[j, i]) * dt
    E = mp.expm(C)
    F = E[0:d, 0:d]
    Q = E[0:d, d:2 * d] * F.T
    return np.array(F.tolist(), dtype=float), np.array(Q.tolist(), dtype=float)


@pytest.mark.parametrize("name", ["rbf6", "quasi1", "per3+m32", "per6+m32", "quasi2", "quasi2+m32"])
@pytest.mark.parametrize("dt", [1e-9, 2.4e-7, 1.22e-4, 1e-3, 0.02, 0.3, 2.5])
def test_kw_discretize_vs_high_precision(cuda_device, name, dt):
    """The per-step discretisation the wide path launches for the model (d > 3, uniform_dt = 0:
    lane-per-row for d <= 8, per-block for block-diagonal d > 8 — per3+m32, per6+m32 in 2 x 2
    blocks, quasi2 in 4 x 4 — else kw_discretize) for one step against a 40-digit Van Loan: F and Q
    to ~1e-13 of their scale and, for small steps, every entry of Q above the rounding level of
    the matrix to relative accuracy (the regime where the stationary shortcut cancels)."""
    m = P.Model(PADE_MODELS[name], 0.05)
    assert m.state_dim > 3
    s = P.pssgp_get_ssm(m.h)
    F, Q = m.discretize(dt)
    Fm, Qm = _mp_van_loan(s["G"], s["W"], dt)
    assert np.max(np.abs(F - Fm)) <= 1e-13 * max(1.0, np.max(np.abs(Fm)))
    assert np.max(np.abs(Q - Qm)) <= 1e-13 * np.max(np.abs(s["Pinf"]))
    if dt <= 0.02:
        big = np.abs(Qm) > 1e-10 * np.max(np.abs(Qm))
        assert np.max(np.abs(Q - Qm)[big] / np.abs(Qm)[big]) <= 1e-10


def test_host_async_pipeline(cuda_device):
    """pssgp_posterior_host_async: several problems in flight on the two internal slots give the
    same results as the synchronous host call, for each problem."""
    m = P.Model([synth.Component("matern52", 1.0, 0.5)], 0.01)
    ws = [synth.random_problem(40 + i, 5000 + 997 * i, kind="matern52", p_missing=0.2, variance=1.0,
                               lengthscale=0.5, noise_var=0.01) for i in range(4)]
    outs = []
    pinned = []
    for w in ws:
        th, yh, mh = (torch.from_numpy(a).pin_memory() for a in (w.t, w.y, w.mask))
        mo = torch.empty(w.N, dtype=torch.float64).pin_memory()
        vo = torch.empty_like(mo)
        no = torch.zeros(1, dtype=torch.float64).pin_memory()
        pinned.append((th, yh, mh))
        outs.append((mo, vo, no))
        P.pssgp_posterior_host_async(m.h, w.N, th, yh, mh, mo, vo, no)
    P.pssgp_sync(m.h)
    for w, (mo, vo, no) in zip(ws, outs):
        mean, var, nll = m.posterior_host(w.t, w.y, w.mask)
        assert np.array_equal(mo.numpy(), mean) and np.array_equal(vo.numpy(), var) and float(no[0]) == float(nll[0])


@pytest.mark.parametrize("case", ["table_rbf3", "pade_rbf3", "wide_pade_rbf6", "wide_table_c4"])
def test_nll_only_all_modes(cuda_device, case):
    """pssgp_nll (no stored state, no smoother; K3's STORE = false instantiation / the wide
    NLL-only path) equals the posterior's NLL and the oracle for every discretisation mode."""
    if case == "table_rbf3":
        w = _uniform([synth.Component("rbf", 1.3, 0.8, order=3)], 0.05, 9001, 0.01, p_missing=0.2, seed=5)
    elif case == "pade_rbf3":
        w = _irregular(PADE_MODELS["rbf3"], 0.05, 9001, seed=6)
    elif case == "wide_pade_rbf6":
        w = _irregular(PADE_MODELS["rbf6"], 0.05, 6001, seed=7)
    else:
        w = synth.config4(n=4096)
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
    t, y, mk = to_dev(w)
    _, _, nll_a = m.posterior(t, y, mk)
    nll_b = m.nll(t, y, mk)
    m.check()
    assert abs(float(nll_a.cpu()[0]) - float(nll_b.cpu()[0])) <= 1e-12 * abs(float(nll_a.cpu()[0]))
    o = oracle.posterior(w, smooth=False)
    assert abs(float(nll_b.cpu()[0]) - o["nll"]) <= NLL_TOL * abs(o["nll"])


def test_cuda_graph_replay(cuda_device):
    """pssgp_posterior captured in a CUDA graph and replayed with new data equals a direct call
    (the K3 carry-publication flag is reset by K1 in stream order, so replays are safe)."""
    w1 = synth.random_problem(50, 30011, kind="matern52", p_missing=0.2, variance=1.0, lengthscale=0.5,
                              noise_var=0.01)
    w2 = synth.random_problem(51, 30011, kind="matern52", p_missing=0.2, variance=1.0, lengthscale=0.5,
                              noise_var=0.01)
    m = P.Model(w1.components, w1.noise_var)
    t, y, mk = to_dev(w1)
    mean = torch.empty_like(t); var = torch.empty_like(t)
    nll = torch.zeros(1, dtype=torch.float64, device="cuda:0")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        m.posterior(t, y, mk, out=(mean, var, nll), stream=s)       # allocate the workspace
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        m.posterior(t, y, mk, out=(mean, var, nll), stream=torch.cuda.current_stream())
    for w in (w2, w1, w2):
        t.copy_(torch.from_numpy(w.t)); y.copy_(torch.from_numpy(w.y)); mk.copy_(torch.from_numpy(w.mask))
        g.replay()
        torch.cuda.synchronize()
        ref = P.Model(w.components, w.noise_var).posterior(*to_dev(w))
        assert torch.equal(mean, ref[0]) and torch.equal(var, ref[1]) and torch.equal(nll, ref[2])


def test_host_async_slot_reuse(cuda_device):
    """Six same-size calls: each slot's device buffers are reused while earlier outputs are still
    draining on the copy-out streams (the input / compute / output event chain)."""
    m = P.Model([synth.Component("matern32", 1.0, 0.5)], 0.02)
    n = 200_000
    ws = [synth.random_problem(70 + i, n, kind="matern32", p_missing=0.2, variance=1.0, lengthscale=0.5,
                               noise_var=0.02) for i in range(6)]
    ins, outs = [], []
    for w in ws:
        th, yh, mh = (torch.from_numpy(a).pin_memory() for a in (w.t, w.y, w.mask))
        mo = torch.empty(n, dtype=torch.float64).pin_memory()
        vo = torch.empty_like(mo)
        no = torch.zeros(1, dtype=torch.float64).pin_memory()
        ins.append((th, yh, mh))
        outs.append((mo, vo, no))
    for (th, yh, mh), (mo, vo, no) in zip(ins, outs):
        P.pssgp_posterior_host_async(m.h, n, th, yh, mh, mo, vo, no)
    P.pssgp_sync(m.h)
    for w, (mo, vo, no) in zip(ws, outs):
        mean, var, nll = m.posterior_host(w.t, w.y, w.mask)
        assert np.array_equal(mo.numpy(), mean) and np.array_equal(vo.numpy(), var) and float(no[0]) == float(nll[0])


@pytest.mark.parametrize("model", ["rbf6", "quasi1"])
def test_wide_quarter_adjoint_rescan_variant(cuda_device, model, tmp_path):
    """The non-default adjoint-form RTS rescan of the quarter path (d <= 8; PSSGP_WIDE_LPR bit 11,
    read once per process, so in a subprocess) against the sequential oracle."""
    import subprocess
    import sys
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
sys.path.insert(0, {os.path.dirname(os.path.abspath(__file__))!r})
import synth, oracle
import paper_2102_09964_b200 as P
from test_gpu_parity import PADE_MODELS, _uniform
comps = PADE_MODELS[{model!r}]
rp = synth.random_problem(7, 3001, kind="matern32", p_missing=0.2)
for w in (_uniform(comps, 0.05, 4001, 0.01, p_missing=0.2, seed=5),
          synth.Workload("jittered", comps, 0.05, rp.t, rp.y, rp.mask)):
    m = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt)
    t, y, mk = (torch.from_numpy(a).cuda() for a in (w.t, w.y, w.mask))
    mean, var, nll = m.posterior(t, y, mk)
    m.check()
    o = oracle.posterior(w)
    em = np.max(np.abs(mean.cpu().numpy() - o["mean"])) / np.max(np.abs(o["mean"]))
    ev = np.max(np.abs(var.cpu().numpy() - o["var"]) / o["var"])
    assert em < 1e-9 and ev < 1e-9, (em, ev)
print("ok")
"""
    env = dict(os.environ, PSSGP_WIDE_LPR="4095")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
