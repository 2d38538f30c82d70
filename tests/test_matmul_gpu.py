"""matmul on the B200: 3xTF32 tcgen05 path within the fp32 bound, exact SIMT
path bit-identical to the reference interpreter (golden) and the oracle."""
import numpy as np
import pytest

from conftest import golden
from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu

U = 2.0 ** -24


def _bound(a, b):
    m = a.shape[1]
    gamma = m * U / (1 - m * U)
    return (2 * gamma + 8 * U) * (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64))


def _within(c, ref, a, b):
    err = np.abs(c.astype(np.float64) - ref.astype(np.float64))
    bound = _bound(a, b)
    worst = float(np.max(err / np.maximum(bound, 1e-300)))
    assert np.all(err <= bound), f"error exceeds (2*gamma_m+8u)|A||B| by x{worst:.3f}"
    return worst


@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (128, 64, 32), (256, 512, 128), (1000, 1000, 1000),
                                   (130, 36, 68), (1, 4, 4)])
def test_matmul_tcgen05_within_fp32_bound(jb, oracle, shape):
    n, m, l = shape
    a, b = W.matmul_inputs(n, m, l, seed=n + m + l)
    c = jb.matmul(a, b)
    ref = oracle.matmul(a, b)
    _within(c, ref, a, b)
    # and much tighter than the bound in practice (3xTF32 ~ fp32)
    rel = np.max(np.abs(c - ref)) / np.max(np.abs(ref))
    assert rel < 1e-5, rel


@pytest.mark.parametrize("tag", ["8x8x8", "5x13x7", "16x16x16"])
def test_matmul_exact_matches_reference_interpreter(jb, tag):
    g = golden("matmul")
    c = jb.matmul(g[f"{tag}_a"], g[f"{tag}_b"], exact=True)
    assert np.array_equal(c.view(np.uint32), g[f"{tag}_res"].view(np.uint32))


def test_matmul_exact_vs_oracle_bitwise(jb, oracle):
    a, b = W.matmul_inputs(300, 257, 129, seed=3)
    c = jb.matmul(a, b, exact=True)
    assert np.array_equal(c.view(np.uint32), oracle.matmul(a, b).view(np.uint32))


def test_matmul_identity_and_zero_k(jb):
    a = np.random.default_rng(1).standard_normal((64, 64)).astype(np.float32)
    eye = np.eye(64, dtype=np.float32)
    np.testing.assert_allclose(jb.matmul(eye, a), a, rtol=1e-6, atol=0)  # truncated-hi 3xTF32: ~2^-21
    z = jb.execute("matmul", [3, 0, 5], [np.zeros((3, 0), np.float32), np.zeros((0, 5), np.float32)])
    assert z.shape == (3, 5) and not z.any()


@pytest.mark.parametrize("shape", [(256, 2048, 256), (1024, 1024, 1024), (128, 4096, 128)])
def test_matmul_deterministic_run_to_run(jb, shape):
    """Split-K slices meet through reductions; with two addends per element
    the result cannot depend on their arrival order: repeated calls are
    bit-identical."""
    n, m, l = shape
    a, b = W.matmul_inputs(n, m, l, seed=7)
    first = jb.matmul(a, b)
    for _ in range(4):
        assert np.array_equal(jb.matmul(a, b).view(np.uint32), first.view(np.uint32))


def test_matmul_graph_replay_and_capture(jb):
    """Repeated calls on the same buffers replay the library's captured graph;
    changing the inputs in place must show up (the graph reads the buffers),
    and a caller's own CUDA-graph capture of the call must work too."""
    import torch
    a, b = W.matmul_inputs(256, 128, 192, seed=3)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c = torch.empty((256, 192), device="cuda")
    from paper_2503_10855_b200 import _lib
    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    outs = []
    for _ in range(3):  # plain, capture on repeat, replay
        assert lib.jb_matmul_f32(256, 128, 192, da.data_ptr(), db.data_ptr(), c.data_ptr(), s) == 0
        outs.append(c.cpu().numpy().copy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    da.mul_(2.0)  # exact scaling: the replay must see the new contents
    assert lib.jb_matmul_f32(256, 128, 192, da.data_ptr(), db.data_ptr(), c.data_ptr(), s) == 0
    np.testing.assert_array_equal(c.cpu().numpy(), outs[0] * 2)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        assert lib.jb_matmul_f32(256, 128, 192, da.data_ptr(), db.data_ptr(), c.data_ptr(), cs.cuda_stream) == 0
    c.zero_()
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(c.cpu().numpy(), outs[0] * 2)
