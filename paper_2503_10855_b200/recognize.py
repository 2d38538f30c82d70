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
from dataclasses import dataclass, field
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
    params: dict = field(default_factory=dict)  # launch parameters the schedule implies


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


# ---------------------------------------------------- scalar-accumulator folds
# ``let s = 0; for k { s += a[i,k]*b[k,j]; } res[i,j] = s;`` and what the
# reduction_tree! macro (fork-chunk, fork-reshape,
# monoid-reassociate, fork-fission) makes of it: the written value is a fold
# (a reduce over a fork, or a loop phi) starting at 0.0 whose term is either
# the product or a read of a partials array, itself written once per thread
# of a "top" fork with the fold of one K chunk (passes/fissfuse.py:134-145).
@dataclass
class _Fold:
    levels: list     # [("fork", f) | ("loop", region)], outermost first: one sequential fold
    term: int        # the summand node
    digits: list     # mixed-radix digits of the fold's iteration, most significant first


def _fold_step(g: _Graph, v):
    """(level, init, body) of a reduce / loop phi."""
    n = g.node(v)
    if n.kind == "reduce" and len(n.inputs) == 2:
        if n.control not in g.fork_of_join:
            raise NotRecognised(f"reduce %{v} hangs off an unmatched join")
        return ("fork", g.fork_of_join[n.control]), n.inputs[0], n.inputs[1]
    if n.kind == "phi" and len(n.inputs) == 2:
        g.loop_induction(n.control)  # a counted loop
        return ("loop", n.control), n.inputs[0], n.inputs[1]
    raise NotRecognised(f"%{v} ({n.kind}) is not a fold")


def _level_digits(g: _Graph, lv) -> list:
    kind, x = lv
    if kind == "fork":
        fk = g.node(x)
        return [(("tid", x, d), int(g.ev(e, g.dcs))) for d, e in enumerate(fk.factors)]
    phi, trip = g.loop_induction(x)
    return [(("loop", x), trip)]


def _is_zero_f32(g: _Graph, i) -> bool:
    n = g.node(i)
    return (n.kind == "constant" and n.const is not None and not n.const.is_zero_collection and
            _scalar_name(n.ty) == "f32" and float(n.const.value) == 0.0)


def _fold(g: _Graph, v) -> _Fold:
    """A sequential f32 sum starting at 0.0: one fold level, or several whose
    inner levels start from the enclosing level's running value (fork-chunk
    without monoid-reassociate)."""
    lv, init, body = _fold_step(g, v)
    if not _is_zero_f32(g, init):
        raise NotRecognised(f"fold %{v} does not start at 0.0")
    levels, cur = [lv], v
    while True:
        b = g.node(body)
        if b.kind == "binary" and b.op == "add" and _scalar_name(b.ty) == "f32" and len(b.inputs) == 2 \
                and list(b.inputs).count(cur) == 1:
            term = b.inputs[0] if b.inputs[1] == cur else b.inputs[1]
            break
        inner_lv, inner_init, inner_body = _fold_step(g, body)  # a carried inner level
        if inner_init != cur:
            raise NotRecognised(f"fold level %{body} does not continue %{cur}")
        levels.append(inner_lv)
        cur, body = body, inner_body
    digits = [d for lv_ in levels for d in _level_digits(g, lv_)]
    return _Fold(levels, term, digits)


def _partials(g: _Graph, arr):
    """A partials array: one reduce over a one-dimensional top fork G whose
    body writes element [tid_G] once from a constant (zero / no-reset)
    collection.  Returns (G, N, inner fold value)."""
    n = g.node(arr)
    if n.kind != "reduce" or n.control not in g.fork_of_join or len(n.inputs) != 2:
        raise NotRecognised(f"partials %{arr} is not a fork reduce")
    G = g.fork_of_join[n.control]
    fk = g.node(G)
    if len(fk.factors) != 1:
        raise NotRecognised(f"top fork %{G} is not one-dimensional")
    N = int(g.ev(fk.factors[0], g.dcs))
    c = g.node(n.inputs[0])
    if c.kind != "constant" or c.const is None or not c.const.is_zero_collection:
        raise NotRecognised(f"partials %{arr} do not start from a constant collection")
    w = g.node(n.inputs[1])
    if w.kind != "write" or w.inputs[0] != arr or len(w.indices) != 1 or len(w.indices[0].ids) != 1:
        raise NotRecognised(f"partials %{arr} are not written once per thread")
    if g.digits(w.indices[0].ids[0]) != [(("tid", G, 0), N)]:
        raise NotRecognised(f"partials %{arr} are not indexed by the top fork's thread")
    return G, N, w.inputs[1]


def _partials_read(g: _Graph, t):
    r = g.node(t)
    if r.kind != "read" or len(r.indices) != 1 or not hasattr(r.indices[0], "ids") or len(r.indices[0].ids) != 1:
        raise NotRecognised(f"term %{t} is neither a product nor a partials read")
    return r.inputs[0], g.digits(r.indices[0].ids[0])


def _product_reads(g: _Graph, t):
    """mul(read P0[x, y], read P1[y', z]) -> (P0 ids, P1 ids)"""
    m_ = g.node(t)
    if m_.kind != "binary" or m_.op != "mul" or _scalar_name(m_.ty) != "f32" or len(m_.inputs) != 2:
        raise NotRecognised(f"term %{t} is not a product")
    by = {}
    for x in m_.inputs:
        r = g.node(x)
        c = g.node(r.inputs[0]) if r.kind == "read" else None
        if c is None or c.kind != "param" or len(r.indices) != 1 or not hasattr(r.indices[0], "ids") \
                or len(r.indices[0].ids) != 2:
            raise NotRecognised(f"product operand %{x} is not a 2-D parameter read")
        by[c.index] = tuple(r.indices[0].ids)
    if set(by) != {0, 1}:
        raise NotRecognised("the product does not read parameters 0 and 1")
    return by[0], by[1]


def _accumulator_form(g: _Graph, value):
    """The written value as a fold tree.  Returns (P0 ids, P1 ids, K digits
    the kernel must see, levels used, tree counts [n1, n2]) where the K
    index is (partition p) * chunk + k' with p = p1 * n2 + p2 folded
    outermost level first."""
    top = _fold(g, value)
    used = list(top.levels)
    if g.node(top.term).kind == "binary":
        a_ids, b_ids = _product_reads(g, top.term)
        return a_ids, b_ids, top.digits, used, [1, 1]
    arr1, idx1 = _partials_read(g, top.term)
    if idx1 != top.digits:
        raise NotRecognised("the bottom fold does not read its own partial")
    G1, N1, v1 = _partials(g, arr1)
    if _span(idx1) != N1:
        raise NotRecognised("the bottom fold does not cover the partials")
    used.append(("fork", G1))
    f1 = _fold(g, v1)
    used += f1.levels
    if g.node(f1.term).kind == "binary":  # one fission: tree [N1]
        a_ids, b_ids = _product_reads(g, f1.term)
        return a_ids, b_ids, [(("tid", G1, 0), N1)] + f1.digits, used, [N1, 1]
    # reduction_tree! applied to the bottom fold again: the middle fold sums
    # partials [q * c + p'] of the deeper array (q = the middle top fork)
    arr2, idx2 = _partials_read(g, f1.term)
    if idx2 != [(("tid", G1, 0), N1)] + f1.digits:
        raise NotRecognised("the middle fold does not read its chunk of the partials")
    G2, N2, v2 = _partials(g, arr2)
    if _span(idx2) != N2:
        raise NotRecognised("the middle folds do not cover the partials")
    used.append(("fork", G2))
    f2 = _fold(g, v2)
    used += f2.levels
    if g.node(f2.term).kind != "binary":
        raise NotRecognised("reduction trees deeper than three layers are not supported")
    a_ids, b_ids = _product_reads(g, f2.term)
    return a_ids, b_ids, [(("tid", G2, 0), N2)] + f2.digits, used, [N1, N2 // N1]


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
    wn = g.node(w.inputs[1])
    if wn.kind in ("reduce", "phi"):
        return _recognise_matmul_acc(g, w, levels)
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
                      f"res[i,j] += a[i,k]*b[k,j] over I={_fmt(wi)} J={_fmt(wj)} K={_fmt(a1)}",
                      {"tile_n": _tile_n(wj), "tree": (1, 1)})


def _check_extents(g: _Graph, n, m, l):
    fn = g.fn
    ev = lambda ty: tuple(int(g.ev(e, g.dcs)) for e in ty.extents)  # noqa: E731
    if len(fn.param_types) != 2:
        raise NotRecognised("matmul takes exactly two parameters")
    pa, pb = fn.param_types[0], fn.param_types[1]
    for ty, want_ext, what in ((pa, (n, m), "a"), (pb, (m, l), "b"), (fn.return_type, (n, l), "result")):
        if type(ty).__name__ != "ArrayType" or ev(ty) != want_ext:
            raise NotRecognised(f"{what} extents differ from the iteration space {want_ext}")
        if _elem(ty) != "f32":
            raise NotRecognised(f"{what} is not f32")


def _tile_n(wj) -> int:
    """CTA tile width from the J axis: the innermost digit of a tiled J
    (fork-tile's inner factor, passes/forks.py:58-62) <= 64 -> 64 columns,
    otherwise (or untiled) 128."""
    return 64 if len(wj) > 1 and wj[-1][1] <= 64 else 128


def _recognise_matmul_acc(g: _Graph, w, coll_levels) -> Recognised:
    """res[i, j] = (fold tree over k of a[i, k] * b[k, j]) written once per
    (i, j): the scalar-accumulator form, plain or as a reduction tree."""
    a_ids, b_ids, kdig, used, tree = _accumulator_form(g, w.inputs[1])
    wi, wj = (g.digits(x) for x in w.indices[0].ids)
    a0, a1 = (g.digits(x) for x in a_ids)
    b0, b1 = (g.digits(x) for x in b_ids)
    if a0 != wi or b1 != wj:
        raise NotRecognised("operand indices are not a[i, .], b[., j] of the written element")
    if a1 != kdig or b0 != kdig:
        raise NotRecognised("the k index is not (partition, chunk offset) of the fold tree "
                            f"(a: {_fmt(a1)}, b: {_fmt(b0)}, tree: {_fmt(kdig)})")
    srcs = [s_ for d in (wi, wj) for s_, _ in d]
    want = set()
    for kind, lv in coll_levels:
        want |= {s_ for s_, _ in _level_digits(g, (kind, lv))}
    if len(srcs) != len(set(srcs)) or set(srcs) != want:
        raise NotRecognised("the write's indices are not the result chain's loop levels")
    ksrcs = [s_ for s_, _ in kdig]
    used_srcs = {s_ for lv in used for s_, _ in _level_digits(g, lv)}
    # every fold level's variable either indexes K or (bottom/middle folds)
    # only selects partials; no level repeats the update
    if len(ksrcs) != len(set(ksrcs)) or not set(ksrcs) <= used_srcs or set(ksrcs) & set(srcs):
        raise NotRecognised("the k index reuses an induction variable")
    n, l, m = _span(wi), _span(wj), _span(kdig)
    _check_extents(g, n, m, l)
    parts = tree[0] * tree[1]
    if parts > 1 and m % parts:
        raise NotRecognised(f"{parts} partials do not divide m = {m}")
    params = {"tile_n": _tile_n(wj), "tree": tuple(tree)}
    return Recognised("matmul", [n, m, l],
                      f"res[i,j] = fold over k of a[i,k]*b[k,j], I={_fmt(wi)} J={_fmt(wj)} K={_fmt(kdig)}, "
                      f"reduction tree {tree[0]}x{tree[1]}", params)


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
