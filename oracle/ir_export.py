"""Serialise a reference (skiff) Module for the C++ IR interpreter.

TEST INFRASTRUCTURE.  ``export_module(module)`` turns the
reference's IR objects (/root/reference/pkg/src/skiff/ir.py:76-286) into one
JSON document that oracle/ir_interp.cpp reads:

  {"functions": {name: {"num_dyn_consts": k, "params": [type...],
                        "ret": type, "nodes": [node | null, ...]}}}

  node  = {"k": kind, "c": control, "i": inputs, "p": preds, "sel": proj
           selection, "f": [dc...] fork factors, "d": thread_id dim,
           "ix": param ordinal, "cv": {"v": literal | null}, "dc": dc,
           "op": operator, "idx": [["P", [ids]] | ["F", n] | ["V", n]],
           "callee": name, "dca": [dc...], "ty": type}
  type  = "f32" | "i64" | "bool" | ... | {"arr": type, "ext": [dc...]}
          | {"prod": [type...]} | {"sum": [type...]}
  dc    = {"p": param index} | {"l": literal} | {"o": "+-*/", "a": dc, "b": dc}

The exporter reads the IR duck-typed; it never executes it.
"""
from __future__ import annotations

import json


def _type(t):
    kind = type(t).__name__
    if kind == "BoolType":
        return "bool"
    if kind == "IntType":
        return f"{'i' if t.signed else 'u'}{t.width}"
    if kind == "FloatType":
        return f"f{t.width}"
    if kind == "ArrayType":
        return {"arr": _type(t.element), "ext": [_dc(e) for e in t.extents]}
    if kind == "ProductType":
        return {"prod": [_type(f) for f in t.fields]}
    if kind == "SummationType":
        return {"sum": [_type(v) for v in t.variants]}
    raise TypeError(f"cannot export type {t!r}")


_DC_OPS = {"DcAdd": "+", "DcSub": "-", "DcMul": "*", "DcDiv": "/"}


def _dc(e):
    kind = type(e).__name__
    if kind == "DcParam":
        return {"p": int(e.index)}
    if kind == "DcLiteral":
        return {"l": int(e.value)}
    return {"o": _DC_OPS[kind], "a": _dc(e.left), "b": _dc(e.right)}


def _literal(v):
    if v is None:
        return None
    if isinstance(v, bool):
        return bool(v)
    if isinstance(v, int):
        return int(v)
    if hasattr(v, "item"):
        v = v.item()
    if isinstance(v, float):
        # repr round-trips the exact double; the interpreter rounds once to
        # the node type, like typed_scalar (values.py:24-31)
        return {"f": repr(float(v))}
    return v


def _index(ix):
    kind = type(ix).__name__
    if kind == "Position":
        return ["P", [int(i) for i in ix.ids]]
    if kind == "Field":
        return ["F", int(ix.ordinal)]
    if kind == "Variant":
        return ["V", int(ix.ordinal)]
    raise TypeError(f"cannot export index {ix!r}")


def _node(n):
    d = {"k": n.kind}
    if n.control is not None:
        d["c"] = int(n.control)
    if n.inputs:
        d["i"] = [int(x) for x in n.inputs]
    if n.preds:
        d["p"] = [int(x) for x in n.preds]
    if n.kind == "proj":
        d["sel"] = int(n.selection)
    if n.kind == "fork":
        d["f"] = [_dc(x) for x in n.factors]
    if n.kind == "thread_id":
        d["d"] = int(n.dim)
    if n.kind == "param":
        d["ix"] = int(n.index)
    if n.kind == "constant":
        d["cv"] = {"v": _literal(n.const.value)}
    if n.kind == "dynconst":
        d["dc"] = _dc(n.dc)
    if n.op:
        d["op"] = n.op
    if n.indices:
        d["idx"] = [_index(ix) for ix in n.indices]
    if n.kind == "call":
        d["callee"] = n.callee
        d["dca"] = [_dc(x) for x in n.dc_args]
    if n.ty is not None:
        d["ty"] = _type(n.ty)
    return d


def export_function(fn) -> dict:
    return {"num_dyn_consts": int(fn.num_dyn_consts),
            "params": [_type(t) for t in fn.param_types],
            "ret": _type(fn.return_type),
            "nodes": [None if n is None else _node(n) for n in fn.nodes]}


def export_module(module) -> str:
    return json.dumps({"functions": {name: export_function(fn) for name, fn in module.functions.items()}},
                      separators=(",", ":"))
