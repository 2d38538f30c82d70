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


def test_fullsize_srad_16384_10_iterations(jb, oracle):
    img = W.srad_image(16384, 16384)
    out, q0 = jb.srad(10, 0.5, img, return_q0sqr=True)
    ref, rq0 = oracle.srad(img, 10, 0.5, return_q0=True)
    assert np.array_equal(_bits(np.asarray(q0)), _bits(np.asarray(rq0)))  # the f64 statistics agree
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)
    assert np.count_nonzero(_bits(out) != _bits(ref)) <= out.size // 10000


def test_fullsize_euler_2048_mesh_10_iterations_bit_exact(jb, oracle):
    areas, nb, normals, ff, v = W.euler_mesh(2048, 2048)
    got = jb.euler(10, areas, nb, normals, ff, v)
    ref = oracle.euler(areas, nb, normals, ff, v, 10)
    assert np.array_equal(_bits(got), _bits(ref))


def test_fullsize_bfs_16m_bit_exact(jb, oracle):
    s, d, e = W.bfs_graph()
    assert np.array_equal(jb.bfs(s, d, e, 0), oracle.bfs(s, d, e, 0))


def test_fullsize_backprop_16m(jb, oracle):
    x, iw, hw, t, ipw, hpw = W.bp_inputs()
    eo, eh, iw2, hw2, ipw2, hpw2 = jb.backprop(x, iw, hw, t, ipw, hpw)
    ref = oracle.bp_train(x, iw, hw, t, ipw, hpw, acc64=True)
    np.testing.assert_allclose(iw2, ref["input_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(ipw2, ref["input_prev_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(hw2, ref["hidden_weights"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose([eo, eh], [ref["out_err"], ref["hid_err"]], rtol=1e-6)
