"""Parity at the benchmark configurations themselves (BASELINE.json configs,
the inputs bench.py times), not only at test sizes: every workload's GPU
result against the oracle restatement on the same full-size inputs.  The
oracle runs multi-threaded on the GPU box's host (a few seconds each)."""
import numpy as np
import pytest

from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _bits(a):
    a = np.ascontiguousarray(a)
    b = a.view(np.uint32).copy()
    b[np.isnan(a)] = 0x7FC00000
    return b


def test_fullsize_edge_batch_256x1080p_bit_exact(jb, oracle):
    g, st, sx, sy, th = W.edge_filters()
    x = W.edge_batch(256, 1080, 1920, seed=1000)
    got = jb.edge_detection(x, g, st, sx, sy, th)
    ref = oracle.edge(x, g, st, sx, sy, th)
    assert np.array_equal(_bits(got), _bits(ref))


def test_fullsize_cava_batch_64x1080p_bit_exact(jb, oracle):
    raw = W.cava_raw(64, 1080, 1920)
    params = W.cava_params(16)
    assert np.array_equal(jb.cava(raw, *params), oracle.cava(raw, *params))


def test_fullsize_matmul_1024_within_fp32_bound(jb, oracle):
    a, b = W.matmul_inputs(1024, 1024, 1024)
    got = jb.matmul(a, b).astype(np.float64)
    ref = oracle.matmul(a, b).astype(np.float64)
    u = 2.0 ** -24
    gam = 1024 * u / (1 - 1024 * u)
    bound = (2 * gam + 8 * u) * (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64))
    assert np.all(np.abs(got - ref) <= bound)


def test_fullsize_srad_16384_10_iterations_exact(jb, oracle):
    img = W.srad_image(16384, 16384)
    out, q0 = jb.srad(10, 0.5, img, return_q0sqr=True, exact=True)
    ref, rq0 = oracle.srad(img, 10, 0.5, return_q0=True)
    assert np.array_equal(_bits(np.asarray(q0)), _bits(np.asarray(rq0)))  # the f64 statistics agree
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)
    assert np.count_nonzero(_bits(out) != _bits(ref)) <= out.size // 10000


def test_fullsize_srad_16384_100_iterations_tolerance(jb, oracle):
    """The timing configuration (niter = 100) in the default
    tolerance mode: rel 1e-4 against the oracle after all iterations."""
    img = W.srad_image(16384, 16384)
    out, q0 = jb.srad(100, 0.5, img, return_q0sqr=True)
    ref, rq0 = oracle.srad(img, 100, 0.5, return_q0=True)
    np.testing.assert_allclose(q0, rq0, rtol=1e-4)
    np.testing.assert_allclose(out, ref, rtol=1e-4, atol=1e-4)


def test_fullsize_euler_2048_mesh_10_iterations_bit_exact(jb, oracle):
    areas, nb, normals, ff, v = W.euler_mesh(2048, 2048)
    got = jb.euler(10, areas, nb, normals, ff, v, exact=True)
    ref = oracle.euler(areas, nb, normals, ff, v, 10)
    assert np.array_equal(_bits(got), _bits(ref))


def test_fullsize_euler_2048_mesh_tolerance(jb, oracle):
    """The default tolerance mode at the benchmark mesh: 1e-5 per RK stage of
    each variable's scale, after 10 iterations (30 stages)."""
    areas, nb, normals, ff, v = W.euler_mesh(2048, 2048)
    got = np.asarray(jb.euler(10, areas, nb, normals, ff, v), np.float64)
    ref = oracle.euler(areas, nb, normals, ff, v, 10).astype(np.float64)
    scale = np.abs(ref).max(axis=1, keepdims=True)
    assert np.all(np.abs(got - ref) <= 1e-5 * 30 * scale)


def test_fullsize_bfs_16m_bit_exact(jb, oracle):
    s, d, e = W.bfs_graph()
    assert np.array_equal(jb.bfs(s, d, e, 0), oracle.bfs(s, d, e, 0))


def test_fullsize_backprop_16m_rodinia_init(jb, oracle):
    """The timed configuration (Rodinia init).  Its hidden sums are ~4e6, so
    squash saturates to 1 and the input-side update is exactly zero: this
    only checks that the step runs and leaves what it must leave; the live
    parity check is the unsaturated test below."""
    x, iw, hw, t, ipw, hpw = W.bp_inputs()
    eo, eh, iw2, hw2, ipw2, hpw2 = jb.backprop(x, iw, hw, t, ipw, hpw)
    ref = oracle.bp_train(x, iw, hw, t, ipw, hpw, acc64=True)
    np.testing.assert_allclose(iw2, ref["input_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(ipw2, ref["input_prev_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(hw2, ref["hidden_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose([eo, eh], [ref["out_err"], ref["hid_err"]], rtol=1e-6)


U = 2.0 ** -24
LAMBDA = 8.0   # probabilistic bound: P(fail) <= 2 exp(-LAMBDA^2 (1-u)^2 / 2) ~ 2.5e-14


def _sum_bound(n_terms, abs_sum):
    """|fl_seq(sum) - fl_64(sum)|: the sequential f32 fold of n terms
    (each an f32 product) differs from the f64-accumulated, once-rounded sum
    by at most the fold's error.  Deterministically that is gamma_{n-1} *
    sum|x_i| (Higham, Thm 4.4), vacuous once n*u >= 1 (n = 2^24 here); we use
    the probabilistic form lambda*sqrt(n)*u*sum|x_i| (Higham & Mary 2019,
    Thm 3.1) plus one rounding of the f64 result."""
    return (LAMBDA * np.sqrt(n_terms) * U + U) * abs_sum


def test_fullsize_backprop_16m_unsaturated(jb, oracle):
    """Every stage live at n_in = 2^24 (weights U(-1,1)*4/sqrt(n), non-zero
    previous weights).  Against the oracle with the GPU's contract (layer
    sums accumulated in f64, rounded once): weights, momenta and errors to
    2 ulp.  Against the reference's own sequential f32 fold
    (oracle acc64=False, pinned to skiff's interpreter by
    tests/golden/bp_*): the hidden units within the stated bound of the
    re-associated sum (squash' <= 1/4)."""
    n = 1 << 24
    x, iw, hw, t, ipw, hpw = W.bp_inputs_unsaturated(n)
    eo, eh, iw2, hw2, ipw2, hpw2, hid, out = jb.backprop(x, iw, hw, t, ipw, hpw, return_layers=True)
    ref64 = oracle.bp_train(x, iw, hw, t, ipw, hpw, acc64=True)
    # the step is live: the input-side weights move
    assert np.count_nonzero(iw2 != iw) > iw.size // 2
    assert np.count_nonzero(ipw2 != ipw) > ipw.size // 2
    for got, want in ((iw2, ref64["input_weights"]), (ipw2, ref64["input_prev_weights"]),
                      (hw2, ref64["hidden_weights"]), (hpw2, ref64["hidden_prev_weights"])):
        ulps = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
        assert ulps.max() <= 2
    np.testing.assert_allclose([eo, eh], [ref64["out_err"], ref64["hid_err"]], rtol=4 * U)
    np.testing.assert_allclose(hid[1:], ref64["hidden"][1:], rtol=4 * U, atol=0)
    # against the sequential f32 fold of the reference interpreter
    seq = oracle.bp_train(x, iw, hw, t, ipw, hpw, acc64=False)
    xs = x.astype(np.float64).copy()
    xs[0] = 1.0
    abs_sum = np.abs(iw.astype(np.float64)).T @ np.abs(xs)
    bound = 0.25 * _sum_bound(n + 1, abs_sum[1:]) + 4 * U
    assert np.all(np.abs(hid[1:].astype(np.float64) - seq["hidden"][1:]) <= bound)
