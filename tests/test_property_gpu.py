"""Randomised parity on the B200 (hypothesis, derandomised so the suite is
reproducible): every kernel family against the oracle restatement on shapes
and data drawn at random -- ragged extents, degenerate sizes, tiles that
straddle frame borders, graphs of every density.  The contracts are the ones
in DESIGN.md §(c): bit-exact for edge, CAVA, CFD and BFS; the fp32 bound
for matmul; q0^2 bit-exact / rel 1e-5 for SRAD."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=40, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])


def _bits(a):
    a = np.ascontiguousarray(a)
    if a.dtype != np.float32:
        return a
    b = a.view(np.uint32).copy()
    b[np.isnan(a)] = 0x7FC00000
    return b


@SETTINGS
@given(b=st.integers(1, 3), n=st.integers(1, 150), m=st.integers(1, 210), seed=st.integers(0, 2**31 - 1),
       theta=st.sampled_from([0.1, 0.0, 0.5, 0.95]))
def test_edge_random_shapes_bit_exact(jb, oracle, b, n, m, seed, theta):
    g, sst, sx, sy, _ = W.edge_filters()
    x = np.stack([W.edge_frame(n, m, seed=seed + k) for k in range(b)])
    th = np.float32(theta)
    got = jb.edge_detection(x, g, sst, sx, sy, th)
    assert np.array_equal(_bits(got), _bits(oracle.edge(x, g, sst, sx, sy, th)))


@SETTINGS
@given(b=st.integers(1, 2), r=st.integers(3, 90), c=st.integers(3, 150), P=st.integers(0, 40),
       seed=st.integers(0, 2**31 - 1))
def test_cava_random_shapes_bit_exact(jb, oracle, b, r, c, P, seed):
    raw = W.cava_raw(b, r, c, seed=seed % 1000)
    tstw, ctrl, wts, coefs, tmap = W.cava_params(P=max(P, 1), seed=seed % 97)
    ctrl, wts = ctrl[:P], wts[:P]
    got = jb.cava(raw, tstw, ctrl, wts, coefs, tmap)
    assert np.array_equal(got, oracle.cava(raw, tstw, ctrl, wts, coefs, tmap))


@SETTINGS
@given(w=st.integers(1, 70), h=st.integers(1, 40), iters=st.integers(1, 3), seed=st.integers(0, 10**6))
def test_euler_random_meshes_bit_exact(jb, oracle, w, h, iters, seed):
    areas, nb, normals, ff, v = W.euler_mesh(w, h, seed=seed)
    got = jb.euler(iters, areas, nb, normals, ff, v, exact=True)
    ref = oracle.euler(areas, nb, normals, ff, v, iters)
    assert np.array_equal(_bits(got), _bits(ref))
    fast = np.asarray(jb.euler(iters, areas, nb, normals, ff, v), np.float64)   # tolerance mode
    scale = np.nanmax(np.abs(ref), axis=1, keepdims=True)
    assert np.all(np.abs(fast - ref) <= 1e-5 * 3 * iters * scale)


@SETTINGS
@given(n=st.integers(1, 3000), maxdeg=st.integers(0, 12), seed=st.integers(0, 10**6), src=st.integers(0, 10**6))
def test_bfs_random_graphs_bit_exact(jb, oracle, n, maxdeg, seed, src):
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, maxdeg + 1, n).astype(np.uint32)
    starting = np.zeros(n, np.uint32)
    np.cumsum(deg[:-1], out=starting[1:])
    edges = rng.integers(0, n, int(deg.sum()), dtype=np.uint32)
    s = src % n
    got = jb.bfs(starting, deg, edges, s)
    assert np.array_equal(got, oracle.bfs(starting, deg, edges, s))


@SETTINGS
@given(n=st.integers(1, 300), m=st.integers(1, 300), l=st.integers(1, 300), seed=st.integers(0, 10**6))
def test_matmul_random_shapes_within_bound(jb, oracle, n, m, l, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (n, m)).astype(np.float32)
    b = rng.uniform(-1, 1, (m, l)).astype(np.float32)
    got = jb.matmul(a, b).astype(np.float64)
    ref = oracle.matmul(a, b).astype(np.float64)
    u = 2.0 ** -24
    gam = m * u / (1 - m * u)
    bound = (2 * gam + 8 * u) * (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64))
    assert np.all(np.abs(got - ref) <= bound + 1e-30)


@SETTINGS
@given(rows=st.integers(2, 140), cols=st.integers(2, 260), niter=st.integers(0, 4), seed=st.integers(0, 10**6))
def test_srad_random_shapes(jb, oracle, rows, cols, niter, seed):
    img = W.srad_image(rows, cols, seed=seed)
    out, q0 = jb.srad(niter, 0.5, img, return_q0sqr=True, exact=True)
    ref, rq0 = oracle.srad(img, niter, 0.5, return_q0=True)
    assert np.array_equal(_bits(np.asarray(q0)), _bits(np.asarray(rq0)))
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)
    fast = jb.srad(niter, 0.5, img)   # tolerance mode (the default)
    np.testing.assert_allclose(fast, ref, rtol=1e-4, atol=1e-4)
