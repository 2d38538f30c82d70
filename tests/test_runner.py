"""Runner (paper_2503_10855_b200/runner.py): one backing arena per device,
reused across calls."""
import numpy as np
import pytest

from paper_2503_10855_b200 import workloads as W
from paper_2503_10855_b200.runner import ALIGN, Runner


def _plan(entry, dcs, args, zero=True):
    r = Runner.__new__(Runner)  # planning needs no device
    r._scratch = {}
    return r.plan(entry, dcs, args, zero)


def test_allocation_plan_is_aligned_and_skips_scalars():
    """Inputs, results and working copies from the dyn-consts and shapes
    alone (sized at invocation), 256-byte aligned."""
    a = np.zeros((3, 5), np.float32)
    b = np.zeros((5, 7), np.float32)
    p = _plan("matmul", [3, 5, 7], [a, b])
    kinds = [(s.kind, s.offset, s.nbytes, s.zero) for s in p.slots]
    assert kinds == [("input", 0, 60, False), ("input", ALIGN, 140, False), ("result", 2 * ALIGN, 84, True),
                     ("scratch", 3 * ALIGN, 0, False)]
    assert p.total == 3 * ALIGN and p.inputs_end == 2 * ALIGN
    s, d, e = W.bfs_graph(64, seed=1)
    p = _plan("bfs", [64, len(e)], [s, d, e, np.uint32(0)])
    assert [x.kind for x in p.slots] == ["input"] * 3 + ["result", "scratch"]
    assert all(x.offset % ALIGN == 0 for x in p.slots)


def test_backprop_plan_separates_working_copies_from_results():
    args = W.bp_inputs(256, 16, 1)
    p = _plan("backprop", [256, 16, 1], list(args))
    kinds = [x.kind for x in p.slots]
    assert kinds == ["input"] * 6 + ["copy"] * 5 + ["result"] * 3 + ["scratch"]
    assert [x.zero for x in p.slots if x.kind == "copy"] == [False] * 5
    assert [x.zero for x in p.slots if x.kind == "result"] == [True] * 3
    assert not any(x.zero for x in _plan("backprop", [256, 16, 1], list(args), zero=False).slots)


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


@pytest.mark.gpu
def test_library_scratch_lives_in_the_runner_arena(jb):
    """The C library's scratch (edge: the packed-gradient ring and its
    control block) is the runner arena's tail once the first call has
    measured it: from the second call on, no allocation and no request the
    bound region cannot hold."""
    g, st, sx, sy, th = W.edge_filters()
    x = np.stack([W.edge_frame(270, 480, seed=s) for s in range(4)])
    r = Runner("edge_detection")
    first = r.run(270, 480, 7, 3, 3, x, g, st, sx, sy, th)
    r.run(270, 480, 7, 3, 3, x, g, st, sx, sy, th)
    allocs, spills = r.stats.allocations, r.stats.scratch_spills
    for _ in range(3):
        got = r.run(270, 480, 7, 3, 3, x, g, st, sx, sy, th)
    assert r.stats.allocations == allocs and r.stats.scratch_spills == spills
    assert r.stats.unplanned == 0
    np.testing.assert_array_equal(got, first)
    np.testing.assert_array_equal(got, jb.edge_detection(x, g, st, sx, sy, th))


@pytest.mark.gpu
def test_module_runner_enforces_the_schedule_and_its_parameters(jb, oracle):
    """A runner over a scheduled module: the schedule's constraint is
    checked at every call (chunk-4 at n = 6: DynConstError naming 4 | n,
    SPEC.md:542-545); a reduction-tree schedule runs with its K partials."""
    skiff = pytest.importorskip("skiff")  # noqa: F841
    import test_schedule_params as T
    from test_dropin_module import CHUNK4, module as mm_module
    from paper_2503_10855_b200.api import DynConstError
    r = Runner("matmul", module=mm_module(schedule=CHUNK4))
    a, b = W.matmul_inputs(8, 8, 8, seed=3)
    np.testing.assert_allclose(r.run(8, 8, 8, a, b), oracle.matmul(a, b), rtol=1e-5, atol=1e-6)
    with pytest.raises(DynConstError, match=r"4 \| n"):
        r.run(6, 8, 8, np.ones((6, 8), np.float32), b)
    rt = Runner("matmul", module=T.module(T.SCHEDULES["tree4"][0]))
    a, b = W.matmul_inputs(256, 512, 128, seed=4)
    got = rt.run(256, 512, 128, a, b)
    assert rt.last_choice.params == {"tile_n": 128, "tree": (4, 1)}
    assert rt.last_choice.c_symbol == "jb_matmul_sched_f32"
    np.testing.assert_array_equal(got, jb.matmul(a, b, tree=(4, 1)))
    np.testing.assert_allclose(got, oracle.matmul(a, b), rtol=1e-4, atol=1e-4)
