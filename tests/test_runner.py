"""Runner (paper_2503_10855_b200/runner.py): one backing arena per device,
reused across calls."""
import numpy as np
import pytest

from paper_2503_10855_b200 import workloads as W
from paper_2503_10855_b200.runner import ALIGN, Runner


def test_allocation_plan_is_aligned_and_skips_scalars():
    a = np.zeros((3, 5), np.float32)
    b = np.zeros(7, np.uint32)
    slots, total = Runner.plan([a, np.float32(0.5), b, 4])
    assert [s[0] for s in slots] == [0, 2]
    assert all(off % ALIGN == 0 for _, off, _ in slots)
    assert slots[1][1] == ALIGN and total == 2 * ALIGN
    assert Runner.plan([])[1] == 0


@pytest.mark.gpu
def test_matmul_runner_reuses_its_arena(jb, oracle):
    r = Runner("matmul")
    a, b = W.matmul_inputs(256, 128, 192, seed=11)
    a0, b0 = a.copy(), b.copy()
    c1 = r.run(256, 128, 192, a, b)
    allocs = r.stats.allocations
    c2 = r.run(256, 128, 192, a, b)
    assert r.stats.allocations == allocs, "same-sized calls must not allocate"
    np.testing.assert_array_equal(c1, c2)
    np.testing.assert_array_equal(c1, jb.matmul(a, b))  # same kernel as the plain API
    assert np.array_equal(a, a0) and np.array_equal(b, b0)  # value semantics
    assert r.stats.copies == [("h2d", 256 * 128 * 4 + 128 * 192 * 4), ("d2h", 256 * 192 * 4)]
    rel = np.max(np.abs(c1 - oracle.matmul(a, b))) / np.max(np.abs(c1))
    assert rel < 1e-5
    # a smaller call fits in the arena; a larger one grows it once
    r.run(64, 64, 64, *W.matmul_inputs(64, 64, 64, seed=1))
    assert r.stats.allocations == allocs
    r.run(512, 512, 512, *W.matmul_inputs(512, 512, 512, seed=2))
    assert r.stats.allocations > allocs


@pytest.mark.gpu
def test_bfs_runner_bit_exact(jb, oracle):
    s, d, e = W.bfs_graph(1 << 14, seed=5)
    r = Runner("bfs")
    got = r.run(len(s), len(e), s, d, e, np.uint32(3))
    np.testing.assert_array_equal(got, oracle.bfs(s, d, e, 3))


@pytest.mark.gpu
def test_srad_and_backprop_runners_match_the_api(jb):
    img = W.srad_image(128, 96, seed=3)
    r = Runner("srad")
    np.testing.assert_array_equal(r.run(128, 96, np.uint64(4), np.float32(0.5), img), jb.srad(4, 0.5, img))
    args = W.bp_inputs(256, 16, 1)
    rb = Runner("backprop")
    got = rb.run(256, 16, 1, *args)
    want = jb.backprop(*args)
    assert len(got) == len(want) == 6
    for g, w in zip(got, want):
        np.testing.assert_array_equal(np.asarray(g), np.asarray(w))


@pytest.mark.gpu
def test_runner_validates_like_execute(jb):
    from paper_2503_10855_b200.api import DynConstError, RuntimeError_
    r = Runner("matmul")
    a, b = W.matmul_inputs(8, 4, 2, seed=0)
    with pytest.raises(RuntimeError_):
        r.run(8, 5, 2, a, b)
    with pytest.raises(DynConstError):
        r.run(8, 4)


@pytest.mark.gpu
def test_edge_runner_batch_matches_api(jb):
    g, st, sx, sy, th = W.edge_filters()
    x = np.stack([W.edge_frame(135, 240, seed=s) for s in range(3)])
    r = Runner("edge_detection")
    got = r.run(135, 240, 7, 3, 3, x, g, st, sx, sy, th)
    np.testing.assert_array_equal(got, jb.edge_detection(x, g, st, sx, sy, th))
    allocs = r.stats.allocations
    r.run(135, 240, 7, 3, 3, x, g, st, sx, sy, th)
    assert r.stats.allocations == allocs
