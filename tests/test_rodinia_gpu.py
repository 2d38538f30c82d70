"""SRAD, CFD/Euler, BFS and backprop on the B200 vs the oracle restatement."""
import numpy as np
import pytest

from conftest import golden
from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _bits(a):
    """Bit patterns, with every NaN mapped to one canonical payload (the
    reference semantics do not distinguish NaN payloads)."""
    a = np.ascontiguousarray(a)
    if a.dtype != np.float32:
        return a
    b = a.view(np.uint32).copy()
    b[np.isnan(a)] = 0x7FC00000
    return b


def _exact(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    assert got.shape == ref.shape and got.dtype == ref.dtype
    bad = np.count_nonzero(_bits(got) != _bits(ref))
    assert bad == 0, f"{bad}/{got.size} differ; max |d| = {np.nanmax(np.abs(got.astype(np.float64) - ref)):.3g}"


# ------------------------------------------------------------------ SRAD
@pytest.mark.parametrize("shape,niter", [((64, 64), 3), ((100, 130), 5), ((257, 129), 4), ((1, 1), 2),
                                         ((33, 260), 1), ((48, 48), 0), ((512, 512), 10), ((700, 1000), 3)])
def test_srad_exact_matches_oracle(jb, oracle, shape, niter):
    img = W.srad_image(*shape, seed=shape[0])
    out, q0 = jb.srad(niter, 0.5, img, return_q0sqr=True, exact=True)
    ref, rq0 = oracle.srad(img, niter, 0.5, return_q0=True)
    if shape == (1, 1):  # zero variance: q0 = 0/0 on both sides
        assert np.isnan(q0).all() == np.isnan(rq0).all()
    else:
        _exact(q0, rq0)  # f64 statistics round to the same f32 q0^2
    # contract: rel 1e-5 (exp/log evaluated in double on both sides)
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5, equal_nan=True)
    # observed: bit-identical
    assert np.count_nonzero(_bits(out) != _bits(ref)) <= out.size // 10000


SRAD_TOL = 1e-4   # the tolerance-mode contract: rel, after niter


@pytest.mark.parametrize("shape,niter", [((64, 64), 3), ((100, 130), 5), ((257, 129), 4), ((1, 1), 2),
                                         ((33, 260), 1), ((48, 48), 0), ((512, 512), 10), ((700, 1000), 3),
                                         ((1024, 2048), 30)])
def test_srad_tolerance_mode_matches_oracle(jb, oracle, shape, niter):
    img = W.srad_image(*shape, seed=shape[0])
    out, q0 = jb.srad(niter, 0.5, img, return_q0sqr=True)
    ref, rq0 = oracle.srad(img, niter, 0.5, return_q0=True)
    np.testing.assert_allclose(out, ref, rtol=SRAD_TOL, atol=SRAD_TOL, equal_nan=True)
    np.testing.assert_allclose(q0, rq0, rtol=SRAD_TOL, equal_nan=True)


def test_srad_tolerance_mode_near_singular_coefficients(jb, oracle):
    """Images whose diffusion coefficients sit on the clamp's singularity
    (1 + (qsqr - q0)/q0den -> 0) and flat regions (zero differences): the
    tolerance kernel must hand those pixels to the exact coefficient."""
    rng = np.random.default_rng(5)
    img = np.full((256, 512), 100.0, np.float32)
    img[::7, ::5] = 255.0
    img[3::11, 2::3] = 1.0
    img += (rng.random(img.shape) < 0.01).astype(np.float32) * 50.0
    out = jb.srad(6, 0.5, img)
    ref = oracle.srad(img, 6, 0.5)
    np.testing.assert_allclose(out, ref, rtol=SRAD_TOL, atol=SRAD_TOL)


def test_srad_iteration_pinned_to_reference_interpreter(jb, oracle):
    """One coefficient+update pass against skiff's oracle_execute: the GPU
    pipeline with niter=1 must reproduce the pinned C iteration."""
    g = golden("srad_iter_10x13")
    _exact(oracle.srad_iter(g["J"], float(g["q0sqr"]), float(g["lam"])), g["out"])


# ------------------------------------------------------------------ CFD
def _mesh(w=64, h=48, seed=0):
    return W.euler_mesh(w, h, seed=seed)


@pytest.mark.parametrize("wh,iters", [((64, 48), 1), ((37, 29), 3), ((256, 128), 2), ((1, 1), 1)])
def test_euler_exact_matches_oracle_bitwise(jb, oracle, wh, iters):
    areas, nb, normals, ff, v = _mesh(*wh, seed=wh[0])
    got = jb.euler(iters, areas, nb, normals, ff, v, exact=True)
    ref = oracle.euler(areas, nb, normals, ff, v, iters)
    _exact(got, ref)
    assert not np.array_equal(got, v)  # the state actually evolved


EULER_TOL = 1e-5  # tolerance mode: per RK stage, relative to each variable's scale


def euler_close(got, ref, stages):
    """|got - ref| <= EULER_TOL * stages * max|ref[v]| for each variable v,
    NaN exactly where the oracle has NaN."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    scale = np.nanmax(np.abs(ref), axis=1, keepdims=True)
    err = np.where(ok, np.abs(got - ref), 0.0)
    worst = (err / (EULER_TOL * stages * scale)).max()
    assert worst <= 1.0, f"worst error {worst:.3g} x the tolerance"


@pytest.mark.parametrize("wh,iters", [((64, 48), 1), ((37, 29), 3), ((256, 128), 2), ((1, 1), 1),
                                      ((512, 512), 10)])
def test_euler_tolerance_mode_matches_oracle(jb, oracle, wh, iters):
    areas, nb, normals, ff, v = _mesh(*wh, seed=wh[0])
    got = jb.euler(iters, areas, nb, normals, ff, v)
    ref = oracle.euler(areas, nb, normals, ff, v, iters)
    euler_close(got, ref, 3 * iters)
    assert not np.array_equal(got, v)


def test_euler_fast_path_fallback_bitwise(jb, oracle):
    """Elements outside the fast division/sqrt range (tiny and huge states,
    zero velocity, zero and negative pressure) take the IEEE recompute in
    euler_rk_kernel; the whole result must stay bit-identical."""
    areas, nb, normals, ff, v = _mesh(64, 48, seed=9)
    v = v.copy()
    n = v.shape[1]
    rng = np.random.default_rng(9)
    idx = rng.choice(n, size=n // 8, replace=False)
    k = len(idx) // 5
    v[0, idx[:k]] *= np.float32(1e-9)                        # tiny density
    v[1:4, idx[k:2 * k]] = 0.0                               # zero velocity: ssq = 0
    v[:, idx[2 * k:3 * k]] *= np.float32(3e7)                # huge state
    v[4, idx[3 * k:4 * k]] = 0.5 * v[0, idx[3 * k:4 * k]] * 1e-3  # pressure below zero
    v[1, idx[4 * k:]] = np.float32(2.0 ** -30)               # subnormal-ish velocity squares
    got = jb.euler(2, areas, nb, normals, ff, v, exact=True)
    ref = oracle.euler(areas, nb, normals, ff, v, 2)
    _exact(got, ref)
    # tolerance mode on the same states: special values recomputed exactly
    euler_close(jb.euler(2, areas, nb, normals, ff, v), ref, 6)


def test_euler_stages_bitwise(jb, oracle):
    areas, nb, normals, ff, v = _mesh(80, 60, seed=3)
    _exact(jb.euler_step_factor(v, areas), oracle.euler_step_factor(v, areas))
    _exact(jb.euler_flux(nb, normals, ff, v), oracle.euler_flux(nb, normals, ff, v))


# ------------------------------------------------------------------ BFS
@pytest.mark.parametrize("name", ["bfs_60", "bfs_200", "bfs_1000"])
def test_bfs_matches_reference_interpreter(jb, name):
    g = golden(name)
    _exact(jb.bfs(g["starting"], g["no_of_edges"], g["edges"], int(g["source"])), g["cost"])


@pytest.mark.parametrize("n,seed", [(1 << 16, 1), (100_003, 2), (1 << 20, 3)])
def test_bfs_random_graph_bitwise(jb, oracle, n, seed):
    s, d, e = W.bfs_graph(n, seed=seed)
    src = seed * 7 % n
    _exact(jb.bfs(s, d, e, src), oracle.bfs(s, d, e, src))


def test_bfs_edge_cases(jb, oracle):
    # isolated source, self loops, unreachable tail, zero-degree nodes
    s = np.array([0, 0, 1, 3, 3], np.uint32)
    d = np.array([0, 1, 2, 0, 1], np.uint32)
    e = np.array([2, 2, 3, 4], np.uint32)
    for src in range(5):
        _exact(jb.bfs(s, d, e, src), oracle.bfs(s, d, e, src))
    one = jb.bfs(np.zeros(1, np.uint32), np.zeros(1, np.uint32), np.zeros(0, np.uint32), 0)
    assert one.tolist() == [0]


@pytest.mark.parametrize("n", [300, 1001])
def test_bfs_deep_chain(jb, oracle, n):
    """A path graph: levels beyond the 254 the level bytes hold go through
    the direct-cost fallback; odd n exercises the unaligned expand tail."""
    s = np.arange(n, dtype=np.uint32)
    d = np.ones(n, np.uint32)
    d[-1] = 0
    e = np.arange(1, n, dtype=np.uint32)
    _exact(jb.bfs(s, d, e, 0), oracle.bfs(s, d, e, 0))
    _exact(jb.bfs(s, d, e, 5), oracle.bfs(s, d, e, 5))


# ------------------------------------------------------------------ backprop
@pytest.mark.parametrize("n_in,n_hid", [(1000, 16), (65536, 16), (4097, 8), (333, 32)])
def test_backprop_matches_oracle(jb, oracle, n_in, n_hid):
    x, iw, hw, t, ipw, hpw = W.bp_inputs(n_in, n_hid, 1, seed=n_in)
    # non-saturated variant: small weights so squash is not flat
    iw = (iw - 0.5) * np.float32(4.0 / np.sqrt(n_in))
    iw = iw.astype(np.float32)
    eo, eh, iw2, hw2, ipw2, hpw2 = jb.backprop(x, iw, hw, t, ipw, hpw)
    ref = oracle.bp_train(x, iw, hw, t, ipw, hpw, acc64=True)
    # f64-accumulated layer sums -> the same f32 with overwhelming probability
    np.testing.assert_allclose(iw2, ref["input_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(hw2, ref["hidden_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(ipw2, ref["input_prev_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(hpw2, ref["hidden_prev_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose([eo, eh], [ref["out_err"], ref["hid_err"]], rtol=1e-6)
    assert np.count_nonzero(_bits(iw2) != _bits(ref["input_weights"])) <= iw2.size // 1000


def test_backprop_adjust_pinned(oracle):
    g = golden("bp_33x5")
    w, _ = oracle.bp_adjust_weights(g["delta"], g["ly"], g["w"], g["oldw"])
    _exact(w[:, 1:], g["adjusted"][:, 1:])


def test_euler_stages_match_fixed_interpreter(jb):
    """The GPU step-factor and flux kernels against skiff's interpreter
    (Appendix A defect fixed, oracle/gen_golden_fixed.py) running the Juno
    step factor and flux around their square roots."""
    g = golden("fixed_interp")
    _exact(jb.euler_step_factor(g["eu_vars"], g["eu_areas"]), g["eu_step_factor"])
    _exact(jb.euler_flux(g["eu_nbrs"], g["eu_normals"], g["eu_ff"], g["eu_vars"]), g["eu_flux"])
