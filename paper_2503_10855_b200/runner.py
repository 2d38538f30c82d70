"""Runner: one backing allocation per device, reused across calls.

SURVEY.md §8(f)2.  The paper's runner "owns allocations
of backing memory" and "only needs to make one allocation per device before
invoking Hercules code"; SPEC.md:538-546 specifies ``run(runner, dyn-consts,
args)``: validate the dynamic constants and shapes, size the backing from
them, copy in, execute, copy out, reuse the allocations across calls.

B200 realisation: the allocation plan is evaluated at invocation from the
entry's dynamic constants and argument shapes (api.ENTRIES).  Every array
argument gets a 256-byte aligned slot in ONE device arena and the same slot
in ONE pinned host staging arena; inputs are staged into pinned memory and
moved with a single host-to-device copy, the kernel runs on device views of
the arena, and results come back through pinned memory into fresh numpy
arrays (value semantics: inputs are never mutated, outputs never alias the
arena).  The arenas only grow, so a steady stream of same-sized calls makes
no allocation after the first; ``stats`` counts allocations and the bytes
moved each way (the copy accounting of SPEC.md:617).

    r = Runner("matmul")
    c = r.run(1024, 1024, 1024, a, b)     # dyn-consts first, then data args
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .api import ENTRIES, DynConstError, RuntimeError_, _torch, validate

ALIGN = 256


@dataclass
class RunnerStats:
    calls: int = 0
    allocations: int = 0     # arena (re)allocations, device + host counted once
    arena_bytes: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    copies: list = field(default_factory=list)  # (direction, bytes) of the last call


class Runner:
    def __init__(self, entry: str, device=None):
        if entry not in ENTRIES:
            raise RuntimeError_(f"no B200 kernel for entry {entry!r}; known: {sorted(ENTRIES)}")
        torch = _torch()
        self.entry = entry
        self.spec = ENTRIES[entry]
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        if self.device.type != "cuda":
            raise RuntimeError_("the runner computes on CUDA devices only (no CPU fallback)")
        self._dev = None    # torch.uint8 device arena
        self._host = None   # torch.uint8 pinned host arena
        self._out = None    # pinned host arena for results
        self.stats = RunnerStats()

    # -------------------------------------------------------------- planning
    @staticmethod
    def plan(args) -> tuple[list, int]:
        """Slots (index, offset, nbytes) of the array arguments, and the total."""
        slots, off = [], 0
        for i, a in enumerate(args):
            if isinstance(a, np.ndarray) and a.ndim > 0:
                slots.append((i, off, a.nbytes))
                off += -(-a.nbytes // ALIGN) * ALIGN
        return slots, off

    def _grow(self, nbytes: int, out_bytes: int = 0):
        torch = _torch()
        if self._dev is None or self._dev.numel() < nbytes:
            cap = max(nbytes, ALIGN)
            self._dev = torch.empty(cap, dtype=torch.uint8, device=self.device)
            self._host = torch.empty(cap, dtype=torch.uint8).pin_memory()
            self.stats.allocations += 1
        if out_bytes and (self._out is None or self._out.numel() < out_bytes):
            self._out = torch.empty(max(out_bytes, ALIGN), dtype=torch.uint8).pin_memory()
            self.stats.allocations += 1
        self.stats.arena_bytes = self._dev.numel() + self._host.numel() + \
            (self._out.numel() if self._out is not None else 0)

    # ------------------------------------------------------------------- run
    def run(self, *values):
        """``run(dyn_consts..., args...)`` -> fresh numpy result(s)."""
        torch = _torch()
        k = len(self.spec.dyn_consts)
        if len(values) < k:
            raise DynConstError(f"{self.entry}: expected {k} dynamic constants {self.spec.dyn_consts}")
        dcs, args = [int(x) for x in values[:k]], [np.asarray(a) if isinstance(a, np.ndarray) else a
                                                  for a in values[k:]]
        validate(self.entry, dcs, args)
        slots, total = self.plan(args)
        self._grow(total)
        host = self._host.numpy()
        for i, off, nb in slots:
            host[off:off + nb] = np.ascontiguousarray(args[i]).reshape(-1).view(np.uint8)
        stream = torch.cuda.current_stream(self.device)
        copies = []
        if total:
            self._dev[:total].copy_(self._host[:total], non_blocking=True)
            copies.append(("h2d", total))
        dev_args = list(args)
        for i, off, nb in slots:
            a = args[i]
            view = self._dev[off:off + nb]
            dev_args[i] = view.view(_torch_of(a.dtype)).view(a.shape)
        with torch.cuda.stream(stream):
            res = self.spec.run(dcs, dev_args)
        outs = list(res) if isinstance(res, tuple) else [res]
        tensors = [o for o in outs if isinstance(o, torch.Tensor)]
        out_bytes = sum(-(-t.numel() * t.element_size() // ALIGN) * ALIGN for t in tensors)
        self._grow(total, out_bytes)
        views, off = [], 0
        for t in tensors:
            nb = t.numel() * t.element_size()
            hv = self._out[off:off + nb]
            hv.copy_(t.contiguous().reshape(-1).view(torch.uint8), non_blocking=True)
            views.append((hv, t))
            off += -(-nb // ALIGN) * ALIGN
        if off:
            copies.append(("d2h", sum(t.numel() * t.element_size() for t in tensors)))
        stream.synchronize()
        result, it = [], iter(views)
        for o in outs:
            if isinstance(o, torch.Tensor):
                hv, t = next(it)
                npdt = _numpy_of(t.dtype)
                arr = hv.numpy().view(npdt).reshape(tuple(t.shape)).copy()
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


def _torch_of(np_dtype):
    from .api import _torch_dtype
    return _torch_dtype(np_dtype)


def _numpy_of(torch_dtype):
    torch = _torch()
    table = {torch.float32: np.float32, torch.int32: np.int32, torch.uint8: np.uint8, torch.float64: np.float64,
             torch.int64: np.int64, torch.uint32: np.uint32}
    return table[torch_dtype]
