"""Launch planner and kernel selector for scheduled Juno modules.

SURVEY.md §8 row a18 / §8(f)1.  The paper's GPU backend turns a function's
fork-join nest into launch dimensions (paper §4.4, /root/reference/PAPER.md:
376-383); the reference specifies it as ``launch_plan(function) ->
LaunchPlan`` but does not implement it.
This module implements that contract over the reference's own IR objects and
connects the result to the hand-written B200 kernels:

  * :func:`fork_nest` takes the fork-join nest from the reference's own
    analysis (skiff/analysis.py:199-312 fork_joins / fork_join_nest /
    reduces_of_join; synthetic factor-1 root for several top-level forks,
    the tree of PAPER.md:376) and classifies each fork's reductions;
  * :func:`launch_plan` sizes the tree bottom-up with the paper's three rules
    and splits the root size into blocks and threads;
  * :func:`select_kernel` checks the function's invocation contract and
    recognises its body structurally (recognize.py) -- never by name or
    signature -- and reports the B200 launch geometry next to the plan;
  * :func:`execute_module` is ``oracle_execute`` for a scheduled module: it
    plans, selects and runs (api.execute), and returns the plan it used.

The IR is the reference's; the reference helpers used (analysis,
dynconst) are imported from the package that built the function, so this
package never imports the reference on its own.

Reduction classes (reduce-node attributes, skiff/ir.py:26-28, inferred by
skiff/passes/attrs.py:174-194 or applied by a schedule):
  * ``parallel_reduce`` on every reduce of the join -> parallel fork;
  * otherwise ``monoid_reduce`` on every remaining reduce -> associative;
  * any reduce with neither -> sequential.
"""
from __future__ import annotations

import importlib
from dataclasses import dataclass, field
from typing import Any, Optional, Sequence

PARALLEL_REDUCE = "parallel_reduce"  # skiff/ir.py:26
MONOID_REDUCE = "monoid_reduce"      # skiff/ir.py:27

BLOCK, THREAD, SEQUENTIAL = "BlockLevel", "ThreadLevel", "Sequential"
PARALLEL, COOPERATIVE, SEQ_REDUCE = "Parallel", "CooperativeTile", "Sequential"
WARP = 32              # CooperativeTile width (fixed at warp width)
B200_SMS = 148
MAX_CTA_THREADS = 1024


class PlanError(Exception):
    """Malformed fork nest (a fork whose token paths reach several joins)."""


# ------------------------------------------------------------ symbolic sizes
# A size is an int, a DynConst tree of the reference, or ('mul'|'max', a, b).
def _dc_eval(e, dcs: Sequence[int]) -> int:
    """Evaluate a reference DynConst under concrete values (semantics of
    skiff/dynconst.py:179-204: exact division, no negative intermediates)."""
    kind = type(e).__name__
    if kind == "DcLiteral":
        return int(e.value)
    if kind == "DcParam":
        if e.index >= len(dcs):
            raise PlanError(f"dynamic-constant parameter #{e.index} not supplied")
        return int(dcs[e.index])
    l, r = _dc_eval(e.left, dcs), _dc_eval(e.right, dcs)
    if kind == "DcAdd":
        return l + r
    if kind == "DcMul":
        return l * r
    if kind == "DcSub":
        if l < r:
            raise PlanError(f"negative dynamic constant {l} - {r}")
        return l - r
    if kind == "DcDiv":
        if r == 0 or l % r:
            raise PlanError(f"inexact dynamic-constant division {l}/{r}")
        return l // r
    raise PlanError(f"unknown dynamic-constant node {kind}")


def _dc_str(e, names: Sequence[str]) -> str:
    kind = type(e).__name__
    if kind == "DcLiteral":
        return str(e.value)
    if kind == "DcParam":
        return names[e.index] if e.index < len(names) else f"#{e.index}"
    op = {"DcAdd": "+", "DcSub": "-", "DcMul": "*", "DcDiv": "/"}.get(kind, "?")
    return f"({_dc_str(e.left, names)} {op} {_dc_str(e.right, names)})"


def size_eval(s, dcs: Sequence[int]) -> int:
    if isinstance(s, int):
        return s
    if isinstance(s, tuple):
        a, b = size_eval(s[1], dcs), size_eval(s[2], dcs)
        return a * b if s[0] == "mul" else max(a, b)
    return _dc_eval(s, dcs)


def size_str(s, names: Sequence[str] = ()) -> str:
    if isinstance(s, int):
        return str(s)
    if isinstance(s, tuple):
        a, b = size_str(s[1], names), size_str(s[2], names)
        return f"{a}*{b}" if s[0] == "mul" else f"max({a}, {b})"
    return _dc_str(s, names)


def _mul(a, b):
    if a == 1:
        return b
    if b == 1:
        return a
    if isinstance(a, int) and isinstance(b, int):
        return a * b
    return ("mul", a, b)


def _max(a, b):
    if isinstance(a, int) and isinstance(b, int):
        return max(a, b)
    if a == b:
        return a
    return ("max", a, b)


def _lit(x):
    """A reference DcLiteral as a plain int (so sizes fold), else as is."""
    return int(x.value) if type(x).__name__ == "DcLiteral" else x


def _product(factors):
    out = 1
    for f in factors:
        out = _mul(out, _lit(f))
    return out


# ------------------------------------------------------------- fork nesting
@dataclass
class Nest:
    """One fork-join of the nest (``fork`` None: the synthetic factor-1 root)."""
    fork: Optional[int]
    join: Optional[int]
    factors: list
    body: set
    children: list = field(default_factory=list)
    reduces: list = field(default_factory=list)  # reduce node ids on the join
    kind: str = "parallel"                         # parallel | associative | sequential

    def walk(self):
        yield self
        for c in self.children:
            yield from c.walk()


def _classify(fn, reduces) -> str:
    kind = "parallel"
    for r in reduces:
        attrs = fn.nodes[r].attributes
        if PARALLEL_REDUCE in attrs:
            continue
        if MONOID_REDUCE in attrs:
            kind = "associative"
        else:
            return "sequential"
    return kind


def _analysis(fn):
    """The reference's own analysis module (the package that built ``fn``)."""
    root = type(fn).__module__.split(".")[0]
    return importlib.import_module(f"{root}.analysis")


def fork_nest(fn) -> Optional[Nest]:
    """Containment tree of ``fn``'s fork-joins, or None without forks.

    Fork/join matching and nesting are the reference's own
    (``analysis.fork_joins`` / ``fork_join_nest`` / ``reduces_of_join``,
    skiff/analysis.py:199-312), so the planner cannot drift from them; this
    adds only each fork's reduction class."""
    an = _analysis(fn)
    try:
        infos = an.fork_joins(fn)
        tree = an.fork_join_nest(fn)
    except Exception as e:  # analysis.AnalysisError: forks that do not nest
        raise PlanError(str(e)) from e
    if tree is None:
        return None

    def conv(t) -> Nest:
        kids = [conv(c) for c in t.children]
        if t.fork is None:
            return Nest(None, None, [], set(), children=kids)
        info = infos[t.fork]
        rs = an.reduces_of_join(fn, info.join)
        return Nest(t.fork, info.join, list(fn.nodes[t.fork].factors), set(info.body_controls), kids,
                    reduces=rs, kind=_classify(fn, rs))

    return conv(tree)


# -------------------------------------------------------------- launch plan
@dataclass
class ForkPlan:
    fork: Optional[int]
    factors: list
    size: Any            # launch size of this subtree (symbolic)
    role: str            # BlockLevel | ThreadLevel | Sequential
    reduction: str       # Parallel | CooperativeTile | Sequential
    kind: str
    children: list = field(default_factory=list)

    def walk(self):
        yield self
        for c in self.children:
            yield from c.walk()


@dataclass
class LaunchPlan:
    function: str
    root: Optional[ForkPlan]
    size: Any            # root launch size, valid for the whole function
    blocks: Any          # block-level part of size
    threads: Any         # thread-level part (per block)
    dc_names: tuple = ()

    def forks(self):
        return list(self.root.walk()) if self.root else []

    def evaluate(self, dyn_consts: Sequence[int]) -> dict:
        """Concrete sizes plus the B200 geometry they map to: CTAs of at most
        1024 threads (whole warps), and waves over the 148 SMs."""
        size = size_eval(self.size, dyn_consts)
        blocks = size_eval(self.blocks, dyn_consts)
        threads = size_eval(self.threads, dyn_consts)
        cta = min(MAX_CTA_THREADS, max(WARP, -(-threads // WARP) * WARP))
        ctas = blocks * max(1, -(-threads // cta))
        return {"size": size, "blocks": blocks, "threads": threads, "cta_threads": cta, "ctas": ctas,
                "waves": round(ctas / B200_SMS, 3)}

    def describe(self) -> str:
        names = self.dc_names
        lines = [f"{self.function}: launch size {size_str(self.size, names)} = "
                 f"{size_str(self.blocks, names)} blocks x {size_str(self.threads, names)} threads"]

        def rec(p, depth):
            tag = "root" if p.fork is None else f"fork %{p.fork}"
            fac = ", ".join(size_str(f, names) for f in p.factors) or "1"
            lines.append(f"{'  ' * depth}{tag} [{fac}] {p.kind}: size {size_str(p.size, names)}, "
                         f"{p.role}, reduction {p.reduction}")
            for c in p.children:
                rec(c, depth + 1)

        if self.root:
            rec(self.root, 1)
        return "\n".join(lines)


def _plan_tree(nd: Nest) -> ForkPlan:
    kids = [_plan_tree(c) for c in nd.children]
    child = 1
    for k in kids:
        child = _max(child, k.size)
    factor = _product(nd.factors)
    if nd.kind == "sequential":
        # rule 1: a sequential reduction makes the fork sequential; its launch
        # size is the largest child's (1 if childless)
        return ForkPlan(nd.fork, nd.factors, child, SEQUENTIAL, SEQ_REDUCE, nd.kind, kids)
    if nd.kind == "associative":
        # rule 2: with its iterations on adjacent threads (approximated, as in
        # SPEC.md:500, by "leaf of the nest") the fork can run as a
        # cooperative reduction with sequential children, or sequentially:
        # the larger launch wins.  Non-leaf associative forks run sequential.
        if not kids:
            return ForkPlan(nd.fork, nd.factors, _max(1, factor), THREAD, COOPERATIVE, nd.kind, kids)
        return ForkPlan(nd.fork, nd.factors, child, SEQUENTIAL, SEQ_REDUCE, nd.kind, kids)
    # rule 3: all reductions parallel -> largest child times the fork factor
    return ForkPlan(nd.fork, nd.factors, _mul(child, factor), THREAD, PARALLEL, nd.kind, kids)


def launch_plan(fn) -> LaunchPlan:
    """Paper §4.4 launch plan of one function (SPEC.md:476 ``launch_plan``).

    Block/thread split: multiple blocks only when the top
    fork-join has parallel reductions only -- its factor becomes the block
    count and its children's size the threads per block; every other fork
    enumerates threads inside one block."""
    nest = fork_nest(fn)
    names = tuple(getattr(fn, "dc_names", ()) or ())
    if nest is None:
        return LaunchPlan(fn.name, None, 1, 1, 1, names)
    root = _plan_tree(nest)
    if nest.kind == "parallel":
        factor = _product(nest.factors) if nest.fork is not None else 1
        child = 1
        for k in root.children:
            child = _max(child, k.size)
        if nest.fork is not None:
            root.role = BLOCK
        return LaunchPlan(fn.name, root, root.size, factor, child, names)
    return LaunchPlan(fn.name, root, root.size, 1, root.size, names)


# ---------------------------------------------------------- kernel selection
# the kernel each entry runs on the B200 and its fixed
# launch geometry: the hand-written kernels size themselves to the machine
# (persistent, SM-count multiples), not to the schedule's fork factors
B200_KERNELS = {
    "matmul": ("jb_matmul_f32", "matmul_tcgen05: 128x128 tcgen05 tiles, split-K 2, one CTA per tile"),
    "edge_detection": ("jb_edge_f32", "edge_fused: persistent, 3 CTAs/SM x 256 threads, 60x60 tiles + in-kernel reject"),
    "cava": ("jb_cava_u8", "cava_kernel: 2 CTAs/SM, TMA u8 boxes, one 32x96 tile per CTA step"),
    "srad": ("jb_srad_f32", "srad_stats + srad_strip: grid = SM multiple, register-window strips"),
    "euler": ("jb_euler_f32", "euler_rk: one thread per element, 3 RK stages"),
    "bfs": ("jb_bfs", "bfs_levels: one cooperative persistent kernel, all levels"),
    "backprop": ("jb_bp_train_f32", "bp_forward + bp_adjust: HBM-streaming GEMV and update"),
}


@dataclass
class KernelChoice:
    entry: str           # B200 entry (api.ENTRIES key)
    c_symbol: str        # libjunob200.so function
    geometry: str        # the B200 kernel's own launch geometry
    matched_by: str      # "structure": the function body was recognised (recognize.py)
    plan: LaunchPlan     # the schedule's §4.4 plan of the function
    dyn_consts: list = field(default_factory=list)   # the entry's dyn-consts
    detail: str = ""
    # launch parameters the schedule implies (recognize.py): matmul's CTA
    # tile width from the J fork's fork-tile factor and the K reduction tree
    # of fork-fission (partials per level), SURVEY.md §8(f)1
    params: dict = field(default_factory=dict)


def select_kernel(module, entry: str, dyn_consts: Sequence[int]) -> KernelChoice:
    """Pick the B200 kernel for ``module.functions[entry]`` under
    ``dyn_consts``.

    The function is held to its invocation contract (constraints, exact
    dynamic-constant evaluation: ``DynConstError``) and then recognised from
    its data graph (recognize.py) -- never by name or type signature.  Raises
    api.UnsupportedError when no kernel computes it."""
    from .api import UnsupportedError, _err, _raise_dc
    from .recognize import check_invocation, recognize
    fns = getattr(module, "functions", None)
    if fns is None or entry not in fns:
        raise KeyError(entry)
    fn = fns[entry]
    plan = launch_plan(fn)
    dcs = check_invocation(fn, dyn_consts, _raise_dc)
    rec, why = recognize(fn, dcs)
    if rec is None:
        raise _err(UnsupportedError, f"no B200 kernel computes function {entry!r}: " +
                   "; ".join(f"not {k} ({v})" for k, v in why.items()))
    sym, geo = B200_KERNELS[rec.entry]
    if rec.entry == "matmul":
        tn, (n1, n2) = rec.params.get("tile_n", 128), rec.params.get("tree", (1, 1))
        if tn != 128 or n1 * n2 > 1:
            sym = "jb_matmul_sched_f32"
            geo = (f"grid (l/{tn}, n/128, {n1 * n2} K partials), 320 threads, 3xTF32 tcgen05 128x{tn} tiles; "
                   f"partials folded {n1}x{n2} in the tree's order (mm_fold_kernel)")
    return KernelChoice(rec.entry, sym, geo, "structure", plan, rec.dyn_consts, rec.detail, dict(rec.params))


def execute_module(module, entry: str, dyn_consts, args, max_steps: int = 50_000_000):
    """``oracle_execute`` for a scheduled module: plan the function, select
    the B200 kernel, run it.  Returns (result, KernelChoice)."""
    from .api import execute
    del max_steps
    choice = select_kernel(module, entry, [int(x) for x in dyn_consts])
    return execute(choice.entry, choice.dyn_consts, args, choice.params), choice
