"""Launch planner (paper §4.4; SPEC.md:476-500 launch_plan) and kernel
selector over the reference's own IR (paper_2503_10855_b200/planner.py).

The IR is built with the reference's skiff package (importable in this
container from /root/reference/pkg/src, or from the installed copy under
baseline/_ref); without it these tests skip.  All but the last run on CPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(os.path.join(p, "skiff")) and p not in sys.path:
        sys.path.append(p)
skiff = pytest.importorskip("skiff")
hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

from skiff.dynconst import DcLiteral, DcParam  # noqa: E402
from skiff.ir import Function, MONOID_REDUCE, PARALLEL_REDUCE, ConstValue  # noqa: E402
from skiff.types import F32  # noqa: E402

from paper_2503_10855_b200 import planner as P  # noqa: E402
from paper_2503_10855_b200.api import UnsupportedError  # noqa: E402

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")


# ------------------------------------------------------------ nest builder
# spec = (factor, kind, [children]); kind in parallel|associative|sequential
def _build(spec, num_dc=0):
    fn = Function("k", num_dc, [], F32, entry=True)
    zero = fn.constant(ConstValue(F32, 0.0))

    def emit(ctl, s):
        factor, kind, kids = s
        fk = fn.fork(ctl, [factor if not isinstance(factor, int) else DcLiteral(factor)])
        c = fk
        for k in kids:
            c = emit(c, k)
        j = fn.join(c)
        tid = fn.thread_id(fk, 0)
        r = fn.reduce(j, zero, tid, ty=F32)
        if kind == "parallel":
            fn.node(r).attributes.add(PARALLEL_REDUCE)
        elif kind == "associative":
            fn.node(r).attributes.add(MONOID_REDUCE)
        return j

    c = fn.start
    for top in (spec if isinstance(spec, list) else [spec]):
        c = emit(c, top)
    fn.return_(c, zero)
    return fn


def _brute(spec) -> int:
    """The three rules, restated independently on the spec tree."""
    if isinstance(spec, list):  # synthetic factor-1 root over several top forks
        return max([1] + [_brute(s) for s in spec])
    factor, kind, kids = spec
    child = max([1] + [_brute(k) for k in kids])
    if kind == "sequential":
        return child
    if kind == "associative":
        return max(1, factor) if not kids else child
    return child * factor


# ---------------------------------------------------- SPEC.md:478-484 examples
def test_sequential_childless_is_1():
    # "fork with sequential reduce, childless -> size 1"
    plan = P.launch_plan(_build((64, "sequential", [])))
    assert plan.evaluate([])["size"] == 1
    assert plan.root.role == P.SEQUENTIAL and plan.root.reduction == P.SEQ_REDUCE


def test_parallel_16_of_32_is_512():
    # "parallel fork factor 16 with parallel child factor 32 -> size 512"
    plan = P.launch_plan(_build((16, "parallel", [(32, "parallel", [])])))
    ev = plan.evaluate([])
    assert ev["size"] == 512
    # top fork parallel only -> blocks; the child enumerates threads
    assert (ev["blocks"], ev["threads"]) == (16, 32)
    assert plan.root.role == P.BLOCK and plan.root.children[0].role == P.THREAD


def test_associative_leaf_64_is_64():
    # "childless associative-reduction fork factor 64 -> max(1, 64) = 64"
    plan = P.launch_plan(_build((64, "associative", [])))
    ev = plan.evaluate([])
    assert ev["size"] == 64 and ev["blocks"] == 1 and ev["threads"] == 64
    assert plan.root.reduction == P.COOPERATIVE  # lowered to a warp reduction


def test_symbolic_factor_and_b200_geometry():
    # fork over a dynamic constant: size stays symbolic until invocation
    plan = P.launch_plan(_build((DcParam(0), "parallel", [(DcParam(1), "parallel", [])]), num_dc=2))
    assert "#0" in plan.describe() or "#1" in plan.describe()
    ev = plan.evaluate([300, 2048])
    assert ev["size"] == 300 * 2048 and ev["blocks"] == 300
    # 2048 threads per block split into 1024-thread CTAs
    assert ev["cta_threads"] == 1024 and ev["ctas"] == 600


def test_multiple_top_forks_get_a_synthetic_root():
    plan = P.launch_plan(_build([(8, "parallel", []), (32, "parallel", [(4, "sequential", [])])]))
    assert plan.root.fork is None
    assert plan.evaluate([])["size"] == 32
    assert plan.evaluate([])["blocks"] == 1


nest = st.recursive(
    st.tuples(st.integers(1, 64), st.sampled_from(["parallel", "associative", "sequential"]), st.just([])),
    lambda kids: st.tuples(st.integers(1, 16), st.sampled_from(["parallel", "associative", "sequential"]),
                           st.lists(kids, min_size=1, max_size=3)),
    max_leaves=8)


@settings(max_examples=150, deadline=None)
@given(st.one_of(nest, st.lists(nest, min_size=2, max_size=3)))
def test_plan_matches_brute_force(spec):
    # plan size(root) = an independent recursion over the rules
    plan = P.launch_plan(_build(spec))
    ev = plan.evaluate([])
    assert ev["size"] == _brute(spec)
    assert ev["blocks"] * ev["threads"] == ev["size"]


# ----------------------------------------------- reference fixture programs
MATMUL = """
#[entry]
fn matmul<n, m, l: usize>(a: f32[n, m], b: f32[m, l]) -> f32[n, l] {
  let res : f32[n, l];
  @outer for i in 0..n {
    @middle for j in 0..l {
      @inner for k in 0..m {
        res[i, j] += a[i, k] * b[k, j];
      }
    }
  }
  return res;
}
"""


def _module(src, schedule):
    from skiff.frontend import parse
    from skiff.lower import lower
    from skiff.schedule import parse_schedule, run_schedule
    mod = lower(parse(src))[0]
    run_schedule(mod, parse_schedule(schedule))
    return mod


def test_matmul_module_plan_and_selection():
    mod = _module(MATMUL, "forkify(*); infer-attributes(*); gpu(matmul);")
    assert mod.functions["matmul"].device == "gpu_sim"
    choice = P.select_kernel(mod, "matmul", [64, 32, 16])
    assert choice.entry == "matmul" and choice.c_symbol == "jb_matmul_f32" and choice.matched_by == "structure"
    assert choice.dyn_consts == [64, 32, 16]
    forks = choice.plan.forks()
    assert forks, choice.plan.describe()
    # the forkified k loop carries res[i,j] += ...: an associative leaf
    leaf = [f for f in forks if not f.children]
    assert all(f.kind in ("associative", "parallel", "sequential") for f in forks)
    assert choice.plan.evaluate([64, 32, 16])["size"] >= 1
    assert leaf


def test_selection_is_structural_not_by_name():
    mod = _module(MATMUL.replace("matmul", "mm"), "forkify(*); infer-attributes(*);")
    choice = P.select_kernel(mod, "mm", [8, 4, 2])
    assert choice.entry == "matmul" and choice.matched_by == "structure"
    assert choice.dyn_consts == [8, 4, 2]


def test_unsupported_function_raises():
    src = """
#[entry]
fn twice<n: usize>(x: f32[n]) -> f32[n] {
  let y : f32[n];
  for i in 0..n { y[i] = x[i] + x[i]; }
  return y;
}
"""
    mod = _module(src, "forkify(*); infer-attributes(*);")
    plan = P.launch_plan(mod.functions["twice"])
    assert plan.evaluate([100])["size"] in (1, 100)
    with pytest.raises(UnsupportedError):
        P.select_kernel(mod, "twice", [100])
    with pytest.raises(KeyError):
        P.select_kernel(mod, "nope", [1])


def test_plans_of_every_golden_fixture_program():
    """Every Juno fixture program of oracle/gen_golden.py plans after the
    reference's own forkify + infer-attributes passes."""
    import re
    src = open(os.path.join(ROOT, "oracle", "gen_golden.py")).read()
    progs = dict(re.findall(r'^([A-Z_]+) = """(.*?)"""', src, re.S | re.M))
    assert len(progs) >= 8
    planned = 0
    for name, text in progs.items():
        mod = _module(text, "forkify(*); infer-attributes(*);")
        for fname, fn in mod.functions.items():
            plan = P.launch_plan(fn)
            assert plan.describe().startswith(fname)
            for f in plan.forks():
                assert f.role in (P.BLOCK, P.THREAD, P.SEQUENTIAL)
            dcs = [7] * fn.num_dyn_consts
            ev = plan.evaluate(dcs)
            assert ev["blocks"] * ev["threads"] == ev["size"] >= 1
            planned += 1
    assert planned >= 14


@pytest.mark.gpu
def test_execute_module_runs_the_selected_kernel(jb, oracle):
    """A scheduled module runs end to end: plan -> select -> B200 kernel,
    checked against the oracle within the fp32 matmul bound."""
    import numpy as np
    from paper_2503_10855_b200 import workloads as W
    mod = _module(MATMUL.replace("matmul", "mm"), "forkify(*); infer-attributes(*); gpu(mm);")
    a, b = W.matmul_inputs(96, 64, 80, seed=5)
    c, choice = P.execute_module(mod, "mm", [96, 64, 80], [a, b])
    assert choice.entry == "matmul" and choice.matched_by == "structure"
    ref = oracle.matmul(a, b)
    u = 2.0 ** -24
    gamma = 64 * u / (1 - 64 * u)
    bound = (2 * gamma + 8 * u) * (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64))
    assert np.all(np.abs(c.astype(np.float64) - ref) <= bound)
