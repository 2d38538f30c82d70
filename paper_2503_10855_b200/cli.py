"""Command line: run Juno entries on the B200 with tensor JSON files.

SURVEY.md §8(f)4; the reference's CLI surface is SPEC.md:568-606 (its
``skiff`` console script, pkg/pyproject.toml:20-21, names a module that is
not in the package).  Only the run side applies to this drop-in -- building
and scheduling stay with the reference:

  python -m paper_2503_10855_b200 entries
  python -m paper_2503_10855_b200 run ENTRY --dc n=4 --dc m=4 --dc l=4 \\
        --input a.json --input b.json [-o out.json | --out-dir DIR]
        [--source prog.jn --schedule prog.sch [--oracle]]
  python -m paper_2503_10855_b200 plan --source prog.jn [--schedule s.sch]
        [--function NAME] [--dc k=v ...]

``run`` reads inputs in the reference's tensor format (tensor_io.py), runs
the entry through api.execute (or, with --source, plans and selects the
kernel for the scheduled function: planner.execute_module), writes the
result in the same format (a tuple result: one file per element,
``out_<i>.json``) and prints one machine-readable metrics line (SPEC.md:584
"metrics on a machine-readable trailer line").  ``run --oracle`` is the
SPEC's A/B switch ("runs the value-semantics interpreter
instead"): the same --source/--schedule module, inputs and output files, but
executed by the reference's own interpreter (skiff.runtime.oracle
.oracle_execute), so ``cmp`` on the two output files is the A/B check.  ``plan`` prints the §4.4
launch plan of each function.  --source/--schedule/plan need the reference's
skiff package importable (they parse Juno with it).

Exit codes: 0 ok, 1 runtime error (RuntimeError_/DynConstError/CUDA),
2 usage error (unknown entry, missing file, bad --dc).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

from . import tensor_io


def _parse_dcs(items, names):
    """--dc name=int (any order) or bare ints (declaration order)."""
    named, pos = {}, []
    for it in items or []:
        if "=" in it:
            k, v = it.split("=", 1)
            named[k.strip()] = int(v)
        else:
            pos.append(int(it))
    if named and pos:
        raise ValueError("mix of named and positional --dc values")
    if pos:
        return pos
    unknown = set(named) - set(names)
    if unknown:
        raise ValueError(f"unknown dynamic constants {sorted(unknown)}; expected {list(names)}")
    missing = [n for n in names if n not in named]
    if missing:
        raise ValueError(f"missing dynamic constants {missing}")
    return [named[n] for n in names]


def _skiff_module(source, schedule):
    try:
        from skiff.frontend import parse
        from skiff.lower import lower
        from skiff.schedule import parse_schedule, run_schedule
    except ImportError as e:  # pragma: no cover - depends on the environment
        raise SystemExit(f"--source needs the reference's skiff package importable: {e}")
    with open(source) as f:
        mod = lower(parse(f.read()))[0]
    if schedule:
        with open(schedule) as f:
            run_schedule(mod, parse_schedule(f.read()))
    return mod


def _write_outputs(result, args) -> list:
    outs = list(result) if isinstance(result, tuple) else [result]
    paths = []
    if len(outs) == 1 and args.output:
        paths = [args.output]
    else:
        d = args.out_dir or "."
        os.makedirs(d, exist_ok=True)
        paths = [os.path.join(d, "out.json" if len(outs) == 1 else f"out_{i}.json") for i in range(len(outs))]
    for v, p in zip(outs, paths):
        tensor_io.dump_tensor(v, p)
    return paths


def cmd_entries(args) -> int:
    from .api import ENTRIES
    for name, e in ENTRIES.items():
        print(f"{name}<{', '.join(e.dyn_consts)}>")
    return 0


def cmd_run(args) -> int:
    from . import _lib, api
    try:
        inputs = [tensor_io.load_tensor(p) for p in args.input or []]
    except (OSError, tensor_io.TensorFormatError, KeyError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    if args.oracle and not args.source:
        print("error: --oracle runs the reference interpreter on a module: it needs --source", file=sys.stderr)
        return 2
    module = _skiff_module(args.source, args.schedule) if args.source else None
    if module is None and args.entry not in api.ENTRIES:
        print(f"error: unknown entry {args.entry!r}; known: {sorted(api.ENTRIES)}", file=sys.stderr)
        return 2
    names = api.ENTRIES[args.entry].dyn_consts if args.entry in api.ENTRIES else \
        tuple(module.functions[args.entry].dc_names) if module and args.entry in module.functions else ()
    try:
        dcs = _parse_dcs(args.dc, names)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    launches0 = _lib.launch_count()
    t0 = time.perf_counter()
    extra = {}
    try:
        if args.oracle:
            result, kernel = _reference_oracle(module, args.entry, dcs, inputs), "skiff.oracle_execute"
        elif module is not None:
            from .planner import execute_module
            result, choice = execute_module(module, args.entry, dcs, inputs)
            kernel = choice.entry
            # the C entry and the launch parameters the schedule implied
            extra = {"c_symbol": choice.c_symbol,
                     "params": {k: list(v) if isinstance(v, tuple) else v for k, v in choice.params.items()}}
        else:
            result = api.execute(args.entry, dcs, inputs)
            kernel = args.entry
    except (api.RuntimeError_, api.DynConstError, api.OracleLimitError, KeyError) as e:
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 1
    wall = (time.perf_counter() - t0) * 1e3
    paths = _write_outputs(result, args)
    h2d = sum(int(np.asarray(x).nbytes) for x in inputs)
    outs = result if isinstance(result, tuple) else (result,)
    d2h = sum(int(np.asarray(x).nbytes) for x in outs)
    print(json.dumps({"entry": args.entry, "kernel": kernel, "dyn_consts": dcs, "wall_ms": round(wall, 3),
                      "gpu_launches": _lib.launch_count() - launches0, "h2d_bytes": h2d, "d2h_bytes": d2h,
                      "outputs": paths, **extra}))
    return 0


def _reference_oracle(module, entry, dcs, inputs):
    """``run --oracle``: the reference's value-semantics interpreter
    (skiff/runtime/oracle.py:28-32) on the same module and inputs.  Its
    exceptions are the reference classes; they are re-raised as the
    drop-in's (which also derive from the reference's, api._err) so both
    arms of the A/B report errors the same way."""
    from skiff.dynconst import DynConstError
    from skiff.runtime.oracle import OracleLimitError, oracle_execute
    from skiff.runtime.values import RuntimeError_
    from . import api
    try:
        return oracle_execute(module, entry, list(dcs), list(inputs))
    except OracleLimitError as e:
        raise api._err(api.OracleLimitError, str(e)) from e
    except DynConstError as e:
        raise api._err(api.DynConstError, str(e)) from e
    except RuntimeError_ as e:
        raise api._err(api.RuntimeError_, str(e)) from e


def cmd_plan(args) -> int:
    from .planner import launch_plan
    module = _skiff_module(args.source, args.schedule)
    fns = [args.function] if args.function else sorted(module.functions)
    for name in fns:
        fn = module.functions[name]
        plan = launch_plan(fn)
        print(plan.describe())
        if args.dc:
            print("  " + json.dumps(plan.evaluate(_parse_dcs(args.dc, tuple(fn.dc_names)))))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2503_10855_b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    sub.add_parser("entries", help="list the B200 entries and their dynamic constants")
    r = sub.add_parser("run", help="run an entry on tensor JSON inputs")
    r.add_argument("entry")
    r.add_argument("--dc", action="append", help="dynamic constant: name=int, or ints in order")
    r.add_argument("--input", action="append", help="tensor JSON file, one per parameter in order")
    r.add_argument("-o", "--output", help="output file (single result)")
    r.add_argument("--out-dir", help="output directory (out.json / out_<i>.json)")
    r.add_argument("--source", help="Juno source: plan + select the kernel for ENTRY (needs skiff)")
    r.add_argument("--schedule", help="schedule applied to --source")
    r.add_argument("--oracle", action="store_true",
                   help="A/B: run --source with the reference's value-semantics interpreter instead (SPEC.md:600)")
    p = sub.add_parser("plan", help="print the paper-§4.4 launch plan of each function (needs skiff)")
    p.add_argument("--source", required=True)
    p.add_argument("--schedule")
    p.add_argument("--function")
    p.add_argument("--dc", action="append")
    args = ap.parse_args(argv)
    if args.cmd == "entries":
        return cmd_entries(args)
    if args.cmd == "run":
        return cmd_run(args)
    return cmd_plan(args)


if __name__ == "__main__":
    sys.exit(main())
