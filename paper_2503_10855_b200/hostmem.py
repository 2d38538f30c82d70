"""Host buffers for the numpy-in / numpy-out path (value semantics, PCIe speed).

The reference boundary takes and returns numpy arrays (oracle.py:28-32).
Pageable numpy memory makes every host<->device copy a staged, blocking one
(the driver bounces it through its own pinned buffer), which halves PCIe
throughput and serialises copies with kernels.  Instead:

* inputs: the caller's array is page-locked IN PLACE with
  ``cudaHostRegister`` the first time it is seen (no staging copy), and the
  registration lives exactly as long as the array that owns the memory (a
  ``weakref.finalize`` unregisters it).  Later calls with the same array pay
  nothing; the DMA engine reads the caller's pages directly.  The total
  registered size is capped (oldest registrations are dropped first);
* outputs: results land in pinned memory from torch's caching host
  allocator and are handed out as numpy arrays that own that memory, so a
  steady stream of calls reuses the same pinned blocks.

Inputs are never written (the copies only read them), and every call
synchronises its stream before returning, so no copy is in flight when the
caller regains the array.
"""
from __future__ import annotations

import threading
import weakref
from collections import OrderedDict

import numpy as np

MIN_BYTES = 1 << 20                 # smaller arrays take a plain copy
CAP_BYTES = 48 << 30                # most host memory registered at once

_lock = threading.Lock()
_regs: "OrderedDict[int, tuple[int, object]]" = OrderedDict()   # ptr -> (nbytes, finalizer)
_total = 0
_disabled = False


def _lib():
    from . import _lib as L
    return L.load()


def _owner(a: np.ndarray):
    """The object that owns ``a``'s memory (root of the .base chain)."""
    o = a
    while isinstance(o, np.ndarray) and o.base is not None:
        o = o.base
    return o


def _unregister(ptr: int) -> None:
    global _total
    with _lock:
        ent = _regs.pop(ptr, None)
        if ent is None:
            return
        _total -= ent[0]
    try:
        _lib().jb_host_unregister(ptr)
    except Exception:  # interpreter shutdown
        pass


def _covered(ptr: int, nbytes: int) -> bool:
    for p, (nb, _) in _regs.items():
        if p <= ptr and ptr + nbytes <= p + nb:
            return True
    return False


def pinned_view(a: np.ndarray):
    """A CPU torch tensor over ``a``'s own memory, page-locked when possible
    (contiguous arrays of at least MIN_BYTES), else a plain view."""
    import torch
    global _total, _disabled
    t = torch.from_numpy(a)
    if _disabled or a.nbytes < MIN_BYTES or not a.flags.c_contiguous:
        return t
    ptr, nbytes = a.ctypes.data, a.nbytes
    with _lock:
        if _covered(ptr, nbytes):
            _regs.move_to_end(next(p for p, (nb, _) in _regs.items() if p <= ptr and ptr + nbytes <= p + nb))
            return t
    owner = _owner(a)
    try:
        fin = weakref.finalize(owner, _unregister, ptr)
    except TypeError:           # owner cannot be weakly referenced: no lifetime hook
        return t
    while True:
        with _lock:
            if _total + nbytes <= CAP_BYTES or not _regs:
                break
            old = next(iter(_regs))
        _regs[old][1]()          # runs _unregister(old)
    from ._lib import JB_EINVAL
    code = _lib().jb_host_register(ptr, nbytes)
    if code != 0:
        fin.detach()
        if code != JB_EINVAL:      # EINVAL: already registered by someone else
            _disabled = True       # e.g. memlock limits: fall back to pageable copies
        return t
    with _lock:
        _regs[ptr] = (nbytes, fin)
        _total += nbytes
    return t


def pinned_empty(shape, torch_dtype):
    """A pinned host tensor from torch's caching host allocator."""
    import torch
    return torch.empty(tuple(int(s) for s in shape), dtype=torch_dtype, pin_memory=True)


def registered_bytes() -> int:
    return _total
