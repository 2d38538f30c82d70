"""Schedules parametrise the kernel.

The reduction_tree! macro (fork-chunk,
fork-reshape, monoid-reassociate, fork-fission) and fork-tile
(passes/forks.py:58-62) change how a scheduled matmul is launched:

* the K reduction tree of fork-fission (partials array f32[N],
  passes/fissfuse.py:134-145) becomes the kernel's K partials, folded in
  the tree's order (``jb_matmul_sched_f32``: n1 x n2 partial levels);
* the J fork's fork-tile factor becomes the CTA tile width (64 / 128).

The scalar-accumulator form (``let s = 0; for k { s += ...; } res[i,j] = s``)
is what reduction_tree! needs; the reference interpreter cannot run it
(SURVEY.md Appendix A.2), so parity is checked against the fixed C++
interpreter of oracle/ (§8(f)3), which can.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(os.path.join(p, "skiff")) and p not in sys.path:
        sys.path.append(p)
skiff = pytest.importorskip("skiff")

from skiff.frontend import parse  # noqa: E402
from skiff.lower import lower  # noqa: E402
from skiff.schedule import parse_schedule, run_schedule  # noqa: E402

from paper_2503_10855_b200 import api  # noqa: E402
from paper_2503_10855_b200 import planner as P  # noqa: E402
from paper_2503_10855_b200.recognize import recognize  # noqa: E402

ACC = """
#[entry]
fn matmul<n, m, l: usize>(a: f32[n, m], b: f32[m, l]) -> f32[n, l] {
  let res : f32[n, l];
  @outer for i in 0..n {
    @middle for j in 0..l {
      let s : f32 = INIT;
      @inner for k in 0..m {
        s += a[i, k] * b[BIDX];
      }
      res[i, j] = s;
    }
  }
  return res;
}
"""
F = "forkify(*); forkify(*); forkify(*); infer-attributes(*); "
RT = ("macro reduction_tree![N](F) { fork-chunk![N](F); let (outer, inner) = fork-reshape[[0], [1]](F); "
      "monoid-reassociate(inner); let (top, bottom) = fork-fission(outer); } ")
# name -> (schedule, expected tree, expected tile_n)
SCHEDULES = {
    "sequential": ("", (1, 1), 128),
    "forkified": (F, (1, 1), 128),
    "chunk4-carried": (F + "fork-chunk![4](matmul@inner);", (1, 1), 128),
    "tree4": (F + RT + "reduction_tree![4](matmul@inner);", (4, 1), 128),
    "tree8": (F + RT + "reduction_tree![8](matmul@inner);", (8, 1), 128),
    "tree4-then-2": (F + RT + "fork-chunk![4](matmul@inner); let (outer, inner) = fork-reshape[[0], [1]]"
                     "(matmul@inner); monoid-reassociate(inner); let (top, bottom) = fork-fission(outer); "
                     "reduction_tree![2](bottom);", (2, 2), 128),
    "tile16-jk": (F + "fork-tile![16](matmul@middle);", (1, 1), 64),
    "tile16-j-tree4": (F + RT + "fork-tile![16](matmul@middle \\ matmul@inner); reduction_tree![4](matmul@inner);",
                       (4, 1), 64),
    "tile128-j": (F + "fork-tile![128](matmul@middle \\ matmul@inner);", (1, 1), 128),
}


def module(schedule="", init="0.0", bidx="k, j"):
    mod = lower(parse(ACC.replace("INIT", init).replace("BIDX", bidx)))[0]
    if schedule:
        run_schedule(mod, parse_schedule(schedule))
    return mod


@pytest.mark.parametrize("name", sorted(SCHEDULES))
def test_schedule_parameters_are_recognised(name):
    sch, tree, tile_n = SCHEDULES[name]
    mod = module(sch)
    rec, why = recognize(mod.functions["matmul"], [256, 256, 256])
    assert rec is not None, why
    assert rec.entry == "matmul" and rec.dyn_consts == [256, 256, 256]
    assert rec.params == {"tile_n": tile_n, "tree": tree}
    choice = P.select_kernel(mod, "matmul", [256, 256, 256])
    assert choice.params == rec.params
    assert choice.c_symbol == ("jb_matmul_f32" if tree == (1, 1) and tile_n == 128 else "jb_matmul_sched_f32")


@pytest.mark.parametrize("init,bidx", [("1.0", "k, j"), ("0.0", "j, k")])
def test_other_folds_are_refused(init, bidx):
    """A fold that does not start at 0, or reads b transposed, is not the
    matmul kernel's computation."""
    mod = module(F + RT + "reduction_tree![4](matmul@inner);", init=init, bidx=bidx)
    rec, why = recognize(mod.functions["matmul"], [16, 16, 16])
    assert rec is None and "matmul" in why
    with pytest.raises(api.UnsupportedError):
        api.oracle_execute(mod, "matmul", [16, 16, 16], [np.ones((16, 16), np.float32)] * 2)


def test_tree_constraint_is_enforced():
    """reduction_tree![4] records 4 | m: m = 6 raises before any launch."""
    mod = module(F + RT + "reduction_tree![4](matmul@inner);")
    with pytest.raises(api.DynConstError):
        api.oracle_execute(mod, "matmul", [4, 6, 4], [np.ones((4, 6), np.float32), np.ones((6, 4), np.float32)])


def test_fixed_interpreter_runs_the_accumulator_schedules():
    """The checker side (CPU): the fixed interpreter runs every schedule of
    this file and agrees with the unscheduled program on integer-valued
    data, where every summation order is exact."""
    from oracle.ir_interp import ir_execute
    rng = np.random.default_rng(5)
    n, m, l = 8, 16, 128
    a = rng.integers(-4, 5, (n, m)).astype(np.float32)
    b = rng.integers(-4, 5, (m, l)).astype(np.float32)
    want = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
    for name, (sch, _, _) in SCHEDULES.items():
        got = ir_execute(module(sch), "matmul", [n, m, l], [a, b])
        assert np.array_equal(got, want), name


def _bound(a, b):
    u = 2.0 ** -24
    m = a.shape[1]
    gamma = m * u / (1 - m * u)
    return (2 * gamma + 8 * u) * (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SCHEDULES))
def test_scheduled_parameters_on_the_gpu(jb, name):
    """The scheduled module runs with its own launch parameters: exact on
    integer data (every partial and fold exact), within the fp32 matmul
    bound of the fixed interpreter on random data."""
    from oracle.ir_interp import ir_execute
    sch, tree, tile_n = SCHEDULES[name]
    mod = module(sch)
    n, m, l = 128, 256, 256
    rng = np.random.default_rng(11)
    ai = rng.integers(-4, 5, (n, m)).astype(np.float32)
    bi = rng.integers(-4, 5, (m, l)).astype(np.float32)
    got = api.oracle_execute(mod, "matmul", [n, m, l], [ai, bi])
    assert np.array_equal(got, (ai.astype(np.float64) @ bi.astype(np.float64)).astype(np.float32))
    a = rng.uniform(-1, 1, (n, m)).astype(np.float32)
    b = rng.uniform(-1, 1, (m, l)).astype(np.float32)
    got = api.oracle_execute(mod, "matmul", [n, m, l], [a, b])
    ref = ir_execute(mod, "matmul", [n, m, l], [a, b], max_steps=2_000_000_000)
    assert np.all(np.abs(got.astype(np.float64) - ref.astype(np.float64)) <= _bound(a, b))


@pytest.mark.gpu
@pytest.mark.parametrize("tile_n,tree,m", [(64, (1, 1), 1024), (128, (4, 1), 1024), (64, (2, 2), 1024),
                                           (128, (8, 1), 1024), (128, (4, 1), 96), (64, (3, 1), 96),
                                           (128, (2, 3), 1020)])
def test_matmul_sched_entry(jb, oracle, tile_n, tree, m):
    """jb_matmul_sched_f32 at full and ragged sizes: tensor-core partials when
    every chunk is whole 32-wide k-blocks, the exact SIMT partials otherwise
    (m = 96 in 4 chunks of 24, m = 1020 in 6 chunks of 170); the fold in the
    tree's order; deterministic run to run."""
    rng = np.random.default_rng(m + tile_n)
    n, l = 1024 if m == 1024 else 200, 1024 if m == 1024 else 260
    a = rng.uniform(-1, 1, (n, m)).astype(np.float32)
    b = rng.uniform(-1, 1, (m, l)).astype(np.float32)
    got = api.matmul(a, b, tile_n=tile_n, tree=tree)
    ref = oracle.matmul(a, b)
    assert np.all(np.abs(got.astype(np.float64) - ref.astype(np.float64)) <= _bound(a, b))
    again = api.matmul(a, b, tile_n=tile_n, tree=tree)
    assert np.array_equal(got.view(np.uint32), again.view(np.uint32))
    if m % (tree[0] * tree[1] * 32):  # SIMT partials: each partial is the oracle's sequential chunk sum
        k = m // (tree[0] * tree[1])
        parts = [oracle.matmul(np.ascontiguousarray(a[:, p * k:(p + 1) * k]), np.ascontiguousarray(b[p * k:(p + 1) * k]))
                 for p in range(tree[0] * tree[1])]
        want = np.zeros((n, l), np.float32)
        for p1 in range(tree[0]):
            t = np.zeros((n, l), np.float32)
            for p2 in range(tree[1]):
                t = (t + parts[p1 * tree[1] + p2]).astype(np.float32)
            want = (want + t).astype(np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
