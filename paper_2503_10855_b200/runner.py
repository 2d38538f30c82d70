"""Runner: one backing allocation per device, reused across calls.

SURVEY.md §8(f)2, SPEC.md:538-546 (``run(runner, dyn-consts, args)``): the
runner validates the call -- for a scheduled module, the schedule's
divisibility constraints, named after their pass (``4 | n``,
dynconst.py:241-253) -- sizes and zeroes its backing memory (except
collections marked NoResetConstant), copies the inputs in, executes, and
copies the outputs out.  The paper's runner "only needs to make one
allocation per device before invoking Hercules code".

B200 realisation.  The allocation plan is evaluated at invocation from the
dynamic constants and argument shapes (api.ENTRIES: argument extents, and the
results / working copies each entry function takes):

    [ inputs | results (zeroed) and working copies | library scratch ]

in ONE device arena, mirrored for the inputs and results by ONE pinned host
staging arena.  Inputs move with a single host-to-device copy; the entry
function runs on device views of the arena, its results and value-semantics
working copies are carved out of it (api._ARENA), and the C library's scratch
is the arena's tail, bound to the stream with ``jb_bind_workspace``; results
come back with a single device-to-host copy into fresh numpy arrays (inputs
are never mutated, outputs never alias the arena).  The scratch size is the
library's high-water mark (``jb_workspace_stats``): the first call of a new
shape learns it, the arena grows once, and steady-state calls make no
allocation at all.  ``stats`` counts allocations, zeroed bytes and the bytes
moved each way (the copy accounting of SPEC.md:617).

    r = Runner("matmul")                       # a benchmark entry, or
    r = Runner("matmul", module=mod)           # a scheduled skiff module
    c = r.run(1024, 1024, 1024, a, b)          # dyn-consts first, then data args
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
import numpy as np

from . import _lib
from .api import ENTRIES, _ARENA, _err, _shape, _torch, _torch_dtype, DynConstError, RuntimeError_, validate

ALIGN = 256


def _up(n: int) -> int:
    return -(-int(n) // ALIGN) * ALIGN


@dataclass
class Slot:
    name: str
    offset: int
    nbytes: int
    kind: str        # "input" | "result" | "copy" | "scratch"
    zero: bool = False


@dataclass
class AllocationPlan:
    slots: list
    total: int
    inputs_end: int      # inputs occupy [0, inputs_end)
    results: tuple       # [lo, hi) of the results and working copies
    scratch: tuple       # [lo, hi) bound as the library's scratch


@dataclass
class RunnerStats:
    calls: int = 0
    allocations: int = 0     # arena (re)allocations, device + host counted once
    arena_bytes: int = 0
    zeroed_bytes: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    scratch_spills: int = 0  # library scratch requests the bound region could not hold
    unplanned: int = 0       # result / copy requests outside the plan (caching allocator)
    copies: list = field(default_factory=list)  # (direction, bytes) of the last call


class Runner:
    def __init__(self, entry: str, device=None, module=None):
        torch = _torch()
        self.module = module
        if module is not None:
            fns = getattr(module, "functions", None)
            if fns is None or entry not in fns:
                raise KeyError(entry)
        elif entry not in ENTRIES:
            raise _err(RuntimeError_, f"no B200 kernel for entry {entry!r}; known: {sorted(ENTRIES)}")
        self.entry = entry
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        if self.device.type != "cuda":
            raise _err(RuntimeError_, "the runner computes on CUDA devices only (no CPU fallback)")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._dev = None    # torch.uint8 device arena
        self._host = None   # torch.uint8 pinned host arena (inputs, then results)
        self._scratch = {}  # (B200 entry, dyn-consts, arg shapes) -> library scratch bytes
        self.stats = RunnerStats()
        self.last_choice = None

    # -------------------------------------------------------------- planning
    def _resolve(self, values):
        """(B200 entry, its dyn-consts, args, launch params, result zeroing)
        for one call; a module is held to its own contract first."""
        if self.module is None:
            spec = ENTRIES[self.entry]
            k = len(spec.dyn_consts)
            if len(values) < k:
                raise _err(DynConstError, f"{self.entry}: expected {k} dynamic constants {spec.dyn_consts}")
            dcs, args = [int(x) for x in values[:k]], list(values[k:])
            dcs, args = validate(self.entry, dcs, args)
            return self.entry, dcs, args, {}, True
        from .planner import select_kernel
        fn = self.module.functions[self.entry]
        k = fn.num_dyn_consts
        if len(values) < k:
            raise _err(DynConstError, f"{self.entry}: expected {k} dynamic constants")
        choice = select_kernel(self.module, self.entry, [int(x) for x in values[:k]])
        self.last_choice = choice
        args = list(values[k:])
        dcs, args = validate(choice.entry, choice.dyn_consts, args)
        return choice.entry, dcs, args, choice.params, _result_needs_zero(fn)

    def plan(self, entry: str, dcs, args, zero_results: bool = True) -> AllocationPlan:
        """The call's allocation plan (offsets in the one arena)."""
        slots, off = [], 0
        for i, a in enumerate(args):
            if isinstance(a, np.ndarray) and a.ndim > 0:
                slots.append(Slot(f"arg{i}", off, a.nbytes, "input"))
                off += _up(a.nbytes)
        inputs_end = off
        reqs = ENTRIES[entry].results(dcs, args)
        n_res = _results_count(entry, dcs, args)
        res_lo = off
        for j, (shape, dt) in enumerate(reqs):
            nb = int(np.prod(shape, dtype=np.int64)) * np.dtype(dt).itemsize
            kind = "result" if j >= len(reqs) - n_res else "copy"
            slots.append(Slot(f"{kind}{j}", off, nb, kind, zero=zero_results and kind == "result"))
            off += _up(nb)
        res = (res_lo, off)
        key = (entry, tuple(dcs), tuple(_shape(a) for a in args if isinstance(a, np.ndarray)))
        sb = _up(self._scratch.get(key, 0))
        slots.append(Slot("scratch", off, sb, "scratch"))
        return AllocationPlan(slots, off + sb, inputs_end, res, (off, off + sb))

    def _grow(self, nbytes: int):
        torch = _torch()
        if self._dev is None or self._dev.numel() < nbytes:
            cap = max(_up(nbytes + (nbytes >> 3)), ALIGN)
            self._dev = None
            self._dev = torch.empty(cap, dtype=torch.uint8, device=self.device)
            self._host = torch.empty(cap, dtype=torch.uint8).pin_memory()
            self.stats.allocations += 1
        self.stats.arena_bytes = self._dev.numel() + self._host.numel()

    # ------------------------------------------------------------------- run
    def run(self, *values):
        """``run(dyn_consts..., args...)`` -> fresh numpy result(s)."""
        torch = _torch()
        entry, dcs, args, params, zero = self._resolve(values)
        args = [np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a for a in args]
        plan = self.plan(entry, dcs, args, zero)
        self._grow(plan.total)
        lib = _lib.load()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            host = self._host.numpy()
            for sl in plan.slots:
                if sl.kind == "input":
                    i = int(sl.name[3:])
                    host[sl.offset:sl.offset + sl.nbytes] = args[i].reshape(-1).view(np.uint8)
            copies = []
            if plan.inputs_end:
                self._dev[:plan.inputs_end].copy_(self._host[:plan.inputs_end], non_blocking=True)
                copies.append(("h2d", plan.inputs_end))
            for sl in plan.slots:  # zero-initialised collections (not NoResetConstant)
                if sl.zero and sl.nbytes:
                    self._dev[sl.offset:sl.offset + sl.nbytes].zero_()
                    self.stats.zeroed_bytes += sl.nbytes
            dev_args = list(args)
            for sl in plan.slots:
                if sl.kind == "input":
                    i = int(sl.name[3:])
                    a = args[i]
                    dev_args[i] = self._dev[sl.offset:sl.offset + sl.nbytes].view(_torch_dtype(a.dtype)).view(a.shape)
            # the entry function's results / working copies come from the plan
            pending = [sl for sl in plan.slots if sl.kind in ("copy", "result")]
            base = self._dev.data_ptr()

            def alloc(shape, np_dtype):
                nb = int(np.prod(shape, dtype=np.int64)) * np.dtype(np_dtype).itemsize
                sl = next((x for x in pending if x.nbytes == nb), None)
                if sl is None:
                    self.stats.unplanned += 1
                    return None  # not in the plan: the caching allocator serves it
                pending.remove(sl)
                return self._dev[sl.offset:sl.offset + nb].view(_torch_dtype(np_dtype)).view(shape)
            s_lo, s_hi = plan.scratch
            sc = ctypes.c_void_p(base + s_lo) if s_hi > s_lo else None
            cs = ctypes.c_void_p(stream.cuda_stream)
            high, spills = ctypes.c_uint64(0), ctypes.c_uint64(0)
            _check(lib.jb_bind_workspace(sc, s_hi - s_lo, cs))
            _ARENA.alloc = alloc
            try:
                res = ENTRIES[entry].run(dcs, dev_args, **params) if params else ENTRIES[entry].run(dcs, dev_args)
                _check(lib.jb_workspace_stats(cs, ctypes.byref(high), ctypes.byref(spills)))
            finally:
                # never leave the arena bound: a later call on this stream
                # could otherwise scribble on it after it is freed or regrown
                _ARENA.alloc = None
                lib.jb_bind_workspace(None, 0, cs)
            key = (entry, tuple(dcs), tuple(_shape(a) for a in args if isinstance(a, np.ndarray)))
            if high.value > self._scratch.get(key, 0):
                self._scratch[key] = int(high.value)  # the next call's plan reserves it
            self.stats.scratch_spills += int(spills.value)
            outs = list(res) if isinstance(res, tuple) else [res]
            tensors = [o for o in outs if isinstance(o, torch.Tensor)]
            # results land in the host arena after the inputs' staging area
            views, off = [], 0
            for t in tensors:
                nb = t.numel() * t.element_size()
                views.append((off, nb, t))
                off += _up(nb)
            if off > self._host.numel():  # results outside the plan: a larger host staging arena
                self._host = torch.empty(_up(off), dtype=torch.uint8).pin_memory()
                self.stats.allocations += 1
            for o, nb, t in views:
                self._host[o:o + nb].copy_(t.contiguous().reshape(-1).view(torch.uint8), non_blocking=True)
            if views:
                copies.append(("d2h", sum(nb for _, nb, _ in views)))
            stream.synchronize()
        result, it = [], iter(views)
        hostn = self._host.numpy()
        for o in outs:
            if isinstance(o, torch.Tensor):
                off, nb, t = next(it)
                arr = hostn[off:off + nb].view(_numpy_of(t.dtype)).reshape(tuple(t.shape)).copy()
                result.append(arr[()] if arr.ndim == 0 else arr)
            else:
                result.append(o)
        self.stats.calls += 1
        self.stats.copies = copies
        for d, nb in copies:
            if d == "h2d":
                self.stats.h2d_bytes += nb
            else:
                self.stats.d2h_bytes += nb
        return tuple(result) if isinstance(res, tuple) else result[0]


def _check(code):
    if code != 0:
        raise _err(RuntimeError_, _lib.last_error())


def _results_count(entry: str, dcs, args) -> int:
    """How many of ENTRIES[entry].results are fresh results (the rest are
    working copies of inputs, which need no zeroing)."""
    return {"euler": 0, "backprop": 3}.get(entry, len(ENTRIES[entry].results(dcs, args)))


def _result_needs_zero(fn) -> bool:
    """The returned collection starts as a zero constant unless the schedule
    marked it NoResetConstant (attrs.py: every read dominated by a write)."""
    for _, n in fn.live_nodes():
        if n.kind == "constant" and n.const is not None and n.const.is_zero_collection:
            if getattr(n, "ty", None) == fn.return_type and "no_reset_constant" in n.attributes:
                return False
    return True


def _numpy_of(torch_dtype):
    torch = _torch()
    table = {torch.float32: np.float32, torch.int32: np.int32, torch.uint8: np.uint8, torch.float64: np.float64,
             torch.int64: np.int64, torch.uint32: np.uint32}
    return table[torch_dtype]
