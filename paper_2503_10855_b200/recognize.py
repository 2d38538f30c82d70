"""Invocation checks and structural recognition of scheduled Juno functions.

``oracle_execute(module, entry, dyn_consts, args)`` hands the drop-in a
reference ``Module``.  Before any kernel runs, the function it names must

1. satisfy its invocation contract, exactly as the reference would enforce
   it: every ``fn.constraints`` entry (``DivisibilityConstraint``,
   /root/reference/pkg/src/skiff/dynconst.py:241-253, recorded by fork-chunk
   / fork-tile at passes/forks.py:44-45) holds, and every fork factor,
   dynamic-constant node and parameter extent evaluates with the reference's
   exact rules (``dynconst.evaluate``, dynconst.py:179-204: inexact division
   and negative intermediates raise ``DynConstError``).
   asks the runner to name the violated constraint (``4 | n``);
2. compute what the selected B200 kernel computes.  :func:`recognize` reads
   the function's data graph -- not its name, not its signature -- and
   returns the benchmark it is, or None.

Recognition (matmul, the one benchmark the reference can express with an
entry signature) is schedule-invariant by construction:

* the returned collection is followed back through its loop-carried phis and
  fork reduces to a zero-initialised constant; exactly one ``write`` lies on
  that chain, so each iteration of every level on the chain updates it once;
* the written value's expression tree must be
  ``add(read(acc, [I, J]), mul(read(P_a, [I, K]), read(P_b, [K, J])))``
  (commutative operands sorted), ``acc`` the collection being written;
* every index is a mixed-radix composition of induction variables --
  thread ids of the chain's forks and counted-loop phis -- built only by
  ``add(mul(x, s), y)`` with ``s`` equal to the span of ``y`` (what
  fork-chunk / fork-tile emit, passes/forks.py:50-62, and reshape permutes),
  so each index enumerates its range exactly once;
* the induction variables split into three disjoint axes I, J (the write's
  indices) and K (the rest), each used with one digit order everywhere, and
  every induction variable of the chain is used (an unused one would repeat
  the update);
* the axis spans equal the parameter and return extents.

Together these give ``res[i, j] = 0 + sum over k of a[i, k] * b[k, j]``, each
product once: the contraction the tcgen05 kernel computes (re-associated,
within the fp32 bound stated in DESIGN.md).  Anything else -- a transpose or
element-wise body with matmul's signature, a reduction-tree (fission) or
outlined schedule, a body with an offset index -- is not recognised and the
caller raises ``UnsupportedError``.

The IR is read duck-typed; reference helpers (``dynconst.evaluate``) are
taken from the package that built the function, so this module never
imports the reference on its own.
"""
from __future__ import annotations

import importlib
from dataclasses import dataclass
from typing import Optional, Sequence

COMMUTATIVE = frozenset({"add", "mul", "min", "max", "eq", "ne", "and", "or", "xor"})


class NotRecognised(Exception):
    """Internal: the function is not the pattern being matched."""


def _ref(fn, sub: str):
    """Submodule ``sub`` of the reference package that built ``fn``."""
    root = type(fn).__module__.split(".")[0]
    return importlib.import_module(f"{root}.{sub}")


# ------------------------------------------------------------ invocation
def check_invocation(fn, dyn_consts: Sequence[int], raise_dc) -> list[int]:
    """Enforce ``fn``'s dynamic-constant contract for one call.

    ``raise_dc(msg, cause)`` raises the caller's DynConstError.  Returns the
    dyn-consts as ints."""
    dcs = [int(x) for x in dyn_consts]
    names = list(getattr(fn, "dc_names", []) or [])
    if len(dcs) != fn.num_dyn_consts:
        raise_dc(f"{fn.name}: expected {fn.num_dyn_consts} dynamic constants, got {len(dcs)}", None)
    for i, v in enumerate(dcs):
        if v < 0:
            nm = names[i] if i < len(names) else f"#{i}"
            raise_dc(f"{fn.name}: dynamic constant {nm} = {v} is negative", None)
    dc = _ref(fn, "dynconst")
    env = ", ".join(f"{names[i] if i < len(names) else '#%d' % i}={v}" for i, v in enumerate(dcs))
    for c in getattr(fn, "constraints", []):
        try:
            ok = c.check(dcs)
        except dc.DynConstError as e:
            raise_dc(f"{fn.name}: constraint {c.describe(names)} (from {c.origin}): {e}", e)
        if not ok:
            raise_dc(f"{fn.name}: divisibility constraint {c.describe(names)} violated under {env} "
                     f"(introduced by {c.origin})", None)
    exprs = []
    for _, n in fn.live_nodes():
        if n.kind == "fork":
            exprs += list(n.factors)
        elif n.kind == "dynconst" and n.dc is not None:
            exprs.append(n.dc)
    for ty in list(fn.param_types) + [fn.return_type]:
        exprs += list(getattr(ty, "extents", []) or [])
    for e in exprs:
        try:
            dc.evaluate(e, dcs)
        except dc.DynConstError as err:
            raise_dc(f"{fn.name}: {err} (evaluating {dc.render(e, names)} under {env})", err)
    return dcs


# ------------------------------------------------------------ recognition
@dataclass
class Recognised:
    entry: str                 # B200 entry (api.ENTRIES key)
    dyn_consts: list           # the entry's dyn-consts, in ITS order
    detail: str


class _Graph:
    def __init__(self, fn, dcs):
        self.fn = fn
        self.dcs = dcs
        self.ev = _ref(fn, "dynconst").evaluate
        self.nodes = dict(fn.live_nodes())
        # join -> fork through the reference's own matching (analysis.py:199-237)
        self.fork_of_join = {info.join: f for f, info in _ref(fn, "analysis").fork_joins(fn).items()}
        self.ifs_by_region = {}
        for i, n in self.nodes.items():
            if n.kind == "if":
                self.ifs_by_region.setdefault(n.control, []).append(i)

    def node(self, i):
        n = self.nodes.get(i)
        if n is None:
            raise NotRecognised(f"dead node %{i}")
        return n

    def scalar_value(self, i) -> int:
        """Concrete value of a dynconst / integer constant node."""
        n = self.node(i)
        if n.kind == "dynconst":
            return int(self.ev(n.dc, self.dcs))
        if n.kind == "constant" and n.const is not None and not n.const.is_zero_collection:
            v = n.const.value
            if isinstance(v, (int,)) or (hasattr(v, "is_integer") and float(v).is_integer()):
                return int(v)
        raise NotRecognised(f"%{i} is not a compile-time integer")

    # a counted loop: phi(region, [0, add(phi, 1)]) with if(region, lt(phi, bound))
    def loop_induction(self, region) -> tuple[int, int]:
        """(induction phi, trip count) of the counted loop headed by region."""
        cands = []
        for i, n in self.nodes.items():
            if n.kind != "phi" or n.control != region or len(n.inputs) != 2:
                continue
            init, back = n.inputs
            b = self.nodes.get(back)
            if b is None or b.kind != "binary" or b.op != "add":
                continue
            other = [x for x in b.inputs if x != i]
            if len(b.inputs) != 2 or len(other) != 1:
                continue
            try:
                if self.scalar_value(init) != 0 or self.scalar_value(other[0]) != 1:
                    continue
            except NotRecognised:
                continue
            for f in self.ifs_by_region.get(region, []):
                cond = self.nodes.get(self.node(f).inputs[0])
                if cond is not None and cond.kind == "binary" and cond.op == "lt" and cond.inputs[0] == i:
                    cands.append((i, self.scalar_value(cond.inputs[1])))
        if len(cands) != 1:
            raise NotRecognised(f"region %{region} is not a counted loop")
        return cands[0]

    def digits(self, i) -> list[tuple]:
        """Index %i as mixed-radix digits [(source, trip), ...], most
        significant first; raises NotRecognised for any other form."""
        n = self.node(i)
        if n.kind == "thread_id":
            fk = self.node(n.control)
            return [(("tid", n.control, n.dim), int(self.ev(fk.factors[n.dim], self.dcs)))]
        if n.kind == "phi":
            phi, trip = self.loop_induction(n.control)
            if phi == i:
                return [(("loop", n.control), trip)]
        if n.kind == "binary" and n.op == "add" and len(n.inputs) == 2:
            for hi, lo in (n.inputs, n.inputs[::-1]):
                h = self.nodes.get(hi)
                if h is None or h.kind != "binary" or h.op != "mul":
                    continue
                for x, s in (h.inputs, h.inputs[::-1]):
                    try:
                        stride = self.scalar_value(s)
                    except NotRecognised:
                        continue
                    try:
                        low = self.digits(lo)
                        high = self.digits(x)
                    except NotRecognised:
                        continue
                    if stride == _span(low):
                        return high + low
        raise NotRecognised(f"index %{i} ({n.kind} {getattr(n, 'op', '')}) is not a composition of "
                            "induction variables")


def _span(digits) -> int:
    out = 1
    for _, t in digits:
        out *= t
    return out


def _chain(g: _Graph, v):
    """Collection chain from the returned value back to its initialiser:
    (writes, zero constant, levels), levels = forks of the chain's reduces and
    loop regions of its phis."""
    writes, consts, levels, seen = set(), set(), set(), set()
    todo = [v]
    while todo:
        i = todo.pop()
        if i in seen:
            continue
        seen.add(i)
        n = g.node(i)
        if n.kind == "write":
            writes.add(i)
            todo.append(n.inputs[0])
        elif n.kind == "reduce":
            if n.control not in g.fork_of_join:
                raise NotRecognised(f"reduce %{i} hangs off an unmatched join")
            levels.add(("fork", g.fork_of_join[n.control]))
            todo += list(n.inputs)
        elif n.kind == "phi":
            levels.add(("loop", n.control))
            todo += list(n.inputs)
        elif n.kind == "constant" and n.const is not None and n.const.is_zero_collection:
            consts.add(i)
        else:
            raise NotRecognised(f"the result chain reaches %{i} ({n.kind})")
    return writes, consts, levels, seen


def _expr(g: _Graph, i, chain, reads):
    n = g.node(i)
    if n.kind == "binary":
        kids = [_expr(g, x, chain, reads) for x in n.inputs]
        if n.op in COMMUTATIVE:
            kids.sort(key=repr)
        return (n.op, _scalar_name(n.ty), *kids)
    if n.kind == "read":
        coll = n.inputs[0]
        c = g.node(coll)
        if coll in chain:
            tag = "ACC"
        elif c.kind == "param":
            tag = f"P{c.index}"
        else:
            raise NotRecognised(f"read %{i} of {c.kind} %{coll}")
        if len(n.indices) != 1 or not hasattr(n.indices[0], "ids"):
            raise NotRecognised(f"read %{i} is not a positional array read")
        reads.append((tag, coll, tuple(n.indices[0].ids)))
        return ("read", tag, len(reads) - 1)
    if n.kind == "constant" and n.const is not None and not n.const.is_zero_collection:
        return ("const", _scalar_name(n.ty), repr(n.const.value))
    raise NotRecognised(f"value node %{i} ({n.kind})")


def _recognise_matmul(g: _Graph) -> Recognised:
    fn = g.fn
    ret = [i for i, n in g.nodes.items() if n.kind == "return"]
    if len(ret) != 1:
        raise NotRecognised("function has no single return")
    v = g.node(ret[0]).inputs[0]
    writes, consts, levels, chain = _chain(g, v)
    if len(writes) != 1 or len(consts) != 1:
        raise NotRecognised(f"{len(writes)} writes / {len(consts)} initialisers on the result chain")
    w = g.node(next(iter(writes)))
    if len(w.indices) != 1 or not hasattr(w.indices[0], "ids") or len(w.indices[0].ids) != 2:
        raise NotRecognised("the write is not a 2-D positional write")
    reads: list = []
    tree = _expr(g, w.inputs[1], chain, reads)
    want = ("add", "f32", ("mul", "f32", ("read", "P0", 1), ("read", "P1", 2)), ("read", "ACC", 0))
    shape = _canon(tree)
    if shape != _canon(want):
        raise NotRecognised(f"written value {tree} is not acc + a*b")
    by_tag = {t: (coll, ids) for t, coll, ids in reads}
    if set(by_tag) != {"ACC", "P0", "P1"} or len(reads) != 3:
        raise NotRecognised("reads are not acc, P0, P1")
    acc_coll, acc_ids = by_tag["ACC"]
    if acc_coll != w.inputs[0]:
        raise NotRecognised("the accumulator read is not the collection being written")
    wi, wj = (g.digits(x) for x in w.indices[0].ids)
    if [g.digits(x) for x in acc_ids] != [wi, wj]:
        raise NotRecognised("the accumulator read and the write index different elements")
    a0, a1 = (g.digits(x) for x in by_tag["P0"][1])
    b0, b1 = (g.digits(x) for x in by_tag["P1"][1])
    if a0 != wi or b1 != wj or a1 != b0:
        raise NotRecognised("operand indices are not a[i, k], b[k, j]")
    axes = {"I": wi, "J": wj, "K": a1}
    srcs = [s for d in axes.values() for s, _ in d]
    if len(srcs) != len(set(srcs)):
        raise NotRecognised("an induction variable indexes two axes")
    # every induction variable of the chain's levels is used exactly once
    want_srcs = set()
    for kind, lv in levels:
        if kind == "fork":
            for d in range(len(g.node(lv).factors)):
                want_srcs.add(("tid", lv, d))
        else:
            want_srcs.add(("loop", lv))
    if set(srcs) != want_srcs:
        raise NotRecognised(f"induction variables {sorted(map(str, want_srcs ^ set(srcs)))} are not the "
                            "update's loop levels (an unused level would repeat it)")
    n, l, m = _span(wi), _span(wj), _span(a1)
    ev = lambda ty: tuple(int(g.ev(e, g.dcs)) for e in ty.extents)  # noqa: E731
    pa, pb = fn.param_types[0], fn.param_types[1]
    for ty, want_ext, what in ((pa, (n, m), "a"), (pb, (m, l), "b"), (fn.return_type, (n, l), "result")):
        if type(ty).__name__ != "ArrayType" or ev(ty) != want_ext:
            raise NotRecognised(f"{what} extents differ from the iteration space {want_ext}")
        if _elem(ty) != "f32":
            raise NotRecognised(f"{what} is not f32")
    if len(fn.param_types) != 2:
        raise NotRecognised("matmul takes exactly two parameters")
    return Recognised("matmul", [n, m, l],
                      f"res[i,j] += a[i,k]*b[k,j] over I={_fmt(wi)} J={_fmt(wj)} K={_fmt(a1)}")


def _canon(t):
    """Expression tree with read ordinals dropped (they depend on DFS order)."""
    if isinstance(t, tuple) and t and t[0] == "read":
        return ("read", t[1])
    if isinstance(t, tuple):
        kids = [_canon(x) for x in t[2:]] if t[0] not in ("const",) else list(t[2:])
        if t[0] in COMMUTATIVE:
            kids.sort(key=repr)
        return (t[0], t[1], *kids)
    return t


def _scalar_name(e) -> str:
    kind = type(e).__name__
    if kind == "FloatType":
        return f"f{e.width}"
    if kind == "IntType":
        return f"{'i' if e.signed else 'u'}{e.width}"
    return kind


def _elem(ty) -> str:
    return _scalar_name(ty.element)


def _fmt(digits) -> str:
    return "x".join(f"{s[0]}%{s[1]}" + (f".{s[2]}" if len(s) > 2 else "") + f"[{t}]" for s, t in digits)


RECOGNISERS = {"matmul": _recognise_matmul}


def recognize(fn, dyn_consts: Sequence[int]) -> tuple[Optional[Recognised], dict]:
    """The B200 benchmark ``fn`` computes under ``dyn_consts`` (already
    checked by :func:`check_invocation`), or None; plus each recogniser's
    reason for rejecting it."""
    g = _Graph(fn, list(dyn_consts))
    why = {}
    for name, rec in RECOGNISERS.items():
        try:
            return rec(g), why
        except NotRecognised as e:
            why[name] = str(e)
    return None, why
