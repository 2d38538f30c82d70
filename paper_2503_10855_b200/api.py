"""Host-side mirror of the reference's execution interface.

The reference executes a Juno entry function with
``oracle_execute(module, entry, dyn_consts, args, max_steps)``
(/root/reference/pkg/src/skiff/runtime/oracle.py:28-32): dynamic constants
in declaration order, then arguments in parameter order, numpy arrays in and
numpy arrays out, value semantics (inputs never mutated, fresh outputs;
oracle.py:119-129).  ``execute``/``oracle_execute`` below keep that contract
for the seven Juno benchmark entries and run them on the B200 through
libjunob200.so.  Per-benchmark functions (``matmul``, ``edge_detection`` ...)
are the same calls without the dyn-const list (they are inferred from the
shapes, like the paper's runner).

Arguments may be numpy arrays (host: copied to the device, result copied
back -- the end-to-end path) or CUDA torch tensors (device-resident: the
result stays on the device).  PyTorch is used only for device memory and
streams; all arithmetic happens in the CUDA kernels.

Errors mirror the reference's classes: ``DynConstError`` for negative or
inconsistent dynamic constants (dynconst.py:16-17,179-204) and
``RuntimeError_`` for shape violations (values.py:20, oracle.py:158-159).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable, Optional, Sequence

import os
import threading

import numpy as np

from . import _lib, hostmem


class RuntimeError_(Exception):
    """Mirror of skiff.runtime.values.RuntimeError_ (values.py:20)."""


class DynConstError(Exception):
    """Mirror of skiff.dynconst.DynConstError (dynconst.py:16-17)."""


class OracleLimitError(RuntimeError_):
    """Mirror of skiff.runtime.oracle.OracleLimitError (never raised: the
    device path has no interpreter step budget)."""


class UnsupportedError(RuntimeError_):
    """The entry/config has no kernel in this build (JB_ENOTSUP), or the
    module's function is not a computation any kernel implements."""


# The reference classes each of ours stands for.  Callers written against
# skiff catch skiff's classes; whenever skiff is loaded in this process the
# drop-in raises a class deriving from BOTH ours and the reference's, so
# ``except skiff.dynconst.DynConstError`` and ``except api.DynConstError``
# both work.  (If skiff is not loaded no caller can name its classes.)
_REF_CLASS = {
    RuntimeError_: ("skiff.runtime.values", "RuntimeError_"),
    DynConstError: ("skiff.dynconst", "DynConstError"),
    OracleLimitError: ("skiff.runtime.oracle", "OracleLimitError"),
    UnsupportedError: ("skiff.runtime.values", "RuntimeError_"),
}
_DUAL: dict = {}


def _err(cls, msg: str) -> Exception:
    """An instance of ``cls`` that is also the reference's class of the same
    role when skiff is loaded."""
    import sys
    mod, name = _REF_CLASS.get(cls, (None, None))
    ref = getattr(sys.modules.get(mod), name, None) if mod else None
    if ref is None or issubclass(cls, ref):
        return cls(msg)
    key = (cls, ref)
    dual = _DUAL.get(key)
    if dual is None:
        dual = type(cls.__name__, (cls, ref), {"__module__": cls.__module__, "__doc__": cls.__doc__})
        _DUAL[key] = dual
    return dual(msg)


def _torch():
    import torch  # deferred: importing the package must not need a GPU
    return torch


def _check(status: int, what: str) -> None:
    if status == _lib.JB_OK:
        return
    msg = f"{what}: {_lib.last_error()}"
    if status == _lib.JB_EINVAL:
        raise _err(RuntimeError_, msg)
    if status == _lib.JB_ENOTSUP:
        raise _err(UnsupportedError, msg)
    raise RuntimeError(msg)


# ----------------------------------------------------------------- marshalling
_NP2TORCH = {}


def _torch_dtype(np_dtype):
    torch = _torch()
    if not _NP2TORCH:
        _NP2TORCH.update({np.dtype(np.float32): torch.float32, np.dtype(np.int32): torch.int32,
                          np.dtype(np.uint8): torch.uint8, np.dtype(np.uint32): torch.uint32,
                          np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64})
    return _NP2TORCH[np.dtype(np_dtype)]


class _Call:
    """Collects device buffers for one call; remembers whether results must
    be copied back to the host (numpy in -> numpy out).

    The call's device is the device of its CUDA tensor arguments (else the
    current one); ``on_device()`` makes it current around the library call,
    since the C library resolves scratch, caches and attributes against the
    current device.  Host (numpy) inputs are page-locked in place and copied
    asynchronously (hostmem.py); host results come back through pinned
    memory, with one stream synchronisation before they are returned."""

    def __init__(self, args, device=None):
        torch = _torch()
        self.host = not any(isinstance(a, torch.Tensor) for a in args)
        if device is None:
            dev = next((a.device for a in args if isinstance(a, torch.Tensor) and a.is_cuda), None)
            device = dev if dev is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise _err(RuntimeError_, "libjunob200 computes on CUDA devices only (no CPU fallback)")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.device)
        self._synced = False

    def on_device(self):
        return _torch().cuda.device(self.device)

    def host_array(self, x, np_dtype, name: str):
        a = np.asarray(x)
        if a.dtype != np.dtype(np_dtype):
            if a.dtype.kind != np.dtype(np_dtype).kind and not (a.dtype.kind in "iu" and
                                                                np.dtype(np_dtype).kind in "iu"):
                raise _err(RuntimeError_, f"{name}: expected {np.dtype(np_dtype).name}, got {a.dtype}")
            a = a.astype(np_dtype)
        a = np.ascontiguousarray(a)
        # uint32 has limited torch support: move the raw bytes as int32
        return a.view(np.int32) if a.dtype == np.uint32 else a

    def dev(self, x, np_dtype, name: str, copy: bool = False):
        torch = _torch()
        want = _torch_dtype(np_dtype)
        if isinstance(x, torch.Tensor):
            if x.dtype != want:
                raise _err(RuntimeError_, f"{name}: expected {np.dtype(np_dtype).name}, got {x.dtype}")
            t = x.to(self.device, non_blocking=True)
            if not t.is_contiguous():
                t = t.contiguous()
            elif copy and t.data_ptr() == x.data_ptr():
                slot = _arena_take(t.shape, np_dtype)   # a runner's working copy
                t = slot.copy_(t) if slot is not None else t.clone()
            return t
        h = hostmem.pinned_view(self.host_array(x, np_dtype, name))
        with torch.cuda.stream(self.stream):
            return h.to(self.device, non_blocking=True)

    def empty(self, shape, np_dtype):
        torch = _torch()
        slot = _arena_take(shape, np_dtype)  # inside Runner.run: the result lives in its arena
        if slot is not None:
            return slot
        return torch.empty(tuple(int(s) for s in shape), dtype=_torch_dtype(np_dtype), device=self.device)

    def out(self, t):
        if not self.host:
            return t
        torch = _torch()
        if t.numel() * t.element_size() < hostmem.MIN_BYTES:
            with torch.cuda.stream(self.stream):
                return t.cpu().numpy()
        h = hostmem.pinned_empty(t.shape, t.dtype)
        with torch.cuda.stream(self.stream):
            h.copy_(t, non_blocking=True)
        self.stream.synchronize()
        return h.numpy()

    @property
    def s(self):
        return self.stream.cuda_stream


def _ptr(t) -> int:
    return t.data_ptr()


def _shape(x) -> tuple:
    return tuple(int(s) for s in x.shape)


def _need(cond: bool, msg: str):
    if not cond:
        raise _err(RuntimeError_, msg)


def _scalar(x, ty=float):
    if hasattr(x, "item"):
        x = x.item()
    return ty(x)


# ---------------------------------------------------------------------- matmul
def matmul(a, b, exact: bool = False, tile_n: int = 128, tree: Sequence[int] = (1, 1)):
    """matmul<n,m,l>(a: f32[n,m], b: f32[m,l]) -> f32[n,l].

    Default: 3xTF32 on tcgen05 tensor cores (fp32 tolerance, the k-reduce is
    re-associated).  ``exact=True``: SIMT kernel in the oracle's k order,
    bit-identical to the reference interpreter.  ``tile_n`` / ``tree`` are a
    schedule's launch parameters (planner.select_kernel): the CTA tile width
    from the J fork's fork-tile factor, and the K reduction tree of
    fork-fission (partial counts per level, outermost first; the partial
    products are folded in that order, jb_matmul_sched_f32)."""
    _need(len(_shape(a)) == 2 and len(_shape(b)) == 2, "matmul: a and b must be 2-D")
    n, m = _shape(a)
    m2, l = _shape(b)
    _need(m == m2, f"matmul: inner extents differ ({m} vs {m2})")
    tree = tuple(int(x) for x in tree) + (1,) * (2 - len(tree))
    _need(len(tree) == 2, "matmul: reduction trees deeper than two partial levels are not supported")
    c = _Call([a, b])
    da, db = c.dev(a, np.float32, "a"), c.dev(b, np.float32, "b")
    out = c.empty((n, l), np.float32)
    lib = _lib.load()
    with c.on_device():
        if exact:
            _check(lib.jb_matmul_exact_f32(n, m, l, _ptr(da), _ptr(db), _ptr(out), c.s), "matmul")
        elif tile_n == 128 and tree == (1, 1):
            _check(lib.jb_matmul_f32(n, m, l, _ptr(da), _ptr(db), _ptr(out), c.s), "matmul")
        else:
            _check(lib.jb_matmul_sched_f32(n, m, l, _ptr(da), _ptr(db), _ptr(out), int(tile_n), tree[0], tree[1],
                                           c.s), "matmul")
    return c.out(out)


# ------------------------------------------------------------------------ edge
def edge_detection(input, gaussian_filter, structure, sx, sy, theta):
    """edge_detection<n,m,gs,sz,sb>(input f32[n,m] | f32[batch,n,m], ...) -> f32.

    A 3-D input is a batch of independent frames (the north star's batched
    edge workload); each frame has its own max-gradient reduction."""
    shp = _shape(input)
    _need(len(shp) in (2, 3), "edge_detection: input must be f32[n,m] or f32[batch,n,m]")
    batch, n, m = (1, *shp) if len(shp) == 2 else shp
    gs, sz, sb = (_shape(x)[0] for x in (gaussian_filter, structure, sx))
    _need(_shape(gaussian_filter) == (gs, gs), "edge_detection: gaussian_filter must be square")
    _need(_shape(structure) == (sz, sz), "edge_detection: structure must be square")
    _need(_shape(sx) == (sb, sb) and _shape(sy) == (sb, sb), "edge_detection: sx/sy must be sb x sb")
    c = _Call([input, gaussian_filter, structure, sx, sy])
    if c.host and len(shp) == 3 and batch > 1:
        # a host batch streams through the device: copies overlap kernels
        x = hostmem.pinned_view(c.host_array(input, np.float32, "input"))
        out = hostmem.pinned_empty(shp, _torch().float32)
        edge_detection_pipelined(x, gaussian_filter, structure, sx, sy, theta, out=out, device=c.device)
        return out.numpy()
    din = c.dev(input, np.float32, "input")
    dg, dst, dsx, dsy = (c.dev(x, np.float32, nm) for x, nm in
                         ((gaussian_filter, "gaussian_filter"), (structure, "structure"), (sx, "sx"),
                          (sy, "sy")))
    out = c.empty(shp, np.float32)
    with c.on_device():
        _check(_lib.load().jb_edge_f32(batch, n, m, gs, sz, sb, _ptr(din), _ptr(dg), _ptr(dst), _ptr(dsx),
                                       _ptr(dsy), _scalar(theta), _ptr(out), c.s), "edge_detection")
    return c.out(out)


# Runner.run's arena (runner.py): while it is active, results and working
# copies of the entry functions are carved out of the runner's one device
# allocation instead of the caching allocator
_ARENA = threading.local()


def _arena_take(shape, np_dtype):
    alloc = getattr(_ARENA, "alloc", None)
    return alloc(tuple(int(x) for x in shape), np_dtype) if alloc is not None else None


_PIPE_CACHE: dict = {}
EXPAND_THREADS = int(os.environ.get("JB_EXPAND_THREADS", "3"))


def _pipelined(x, out, chunk: int, key, launch, dev, out_elem=None, finish=None):
    """Host-buffer batch through the device with copy/compute overlap.

    Frames of the host batch ``x`` move in chunks through two device slots on
    three streams -- H2D of chunk i+1 and D2H of chunk i-1 overlap the kernel
    of chunk i -- so a call is bound by the slower PCIe direction instead of
    the sum of copy and compute time.  ``launch(k, din, dout, stream)`` runs
    the entry on the first k frames of the slot buffers.

    By default the device result of a chunk is copied into ``out`` directly.
    With ``out_elem = (shape, torch dtype)`` and ``finish`` the device slots
    hold that per-frame result instead; it lands in one of two pinned host
    staging slots and ``finish(f0, k, staged)`` turns it into ``out[f0:f0+k]``
    on the host, one chunk behind the device (so the host work of chunk i-1
    overlaps the copies and kernel of chunk i)."""
    torch = _torch()
    B = int(x.shape[0])
    e_shape, e_dtype = out_elem if out_elem is not None else (tuple(out.shape[1:]), out.dtype)
    key = (dev.index, x.dtype, tuple(x.shape[1:]), e_dtype, tuple(e_shape), chunk, key)
    st = _PIPE_CACHE.get(key)
    if st is None:
        st = dict(inb=[torch.empty((chunk, *x.shape[1:]), dtype=x.dtype, device=dev) for _ in range(2)],
                  outb=[torch.empty((chunk, *e_shape), dtype=e_dtype, device=dev) for _ in range(2)],
                  stage=[hostmem.pinned_empty((chunk, *e_shape), e_dtype) for _ in range(2)]
                  if finish is not None else None,
                  s_in=torch.cuda.Stream(dev), s_out=torch.cuda.Stream(dev))
        _PIPE_CACHE[key] = st
    comp = torch.cuda.current_stream(dev)
    s_in, s_out = st["s_in"], st["s_out"]
    c_done = [None, None]
    d_done = [None, None]
    pending = None  # (f0, k, slot, event) of the chunk whose host finish is due
    for i, f0 in enumerate(range(0, B, chunk)):
        k = min(chunk, B - f0)
        slot = i & 1
        din, dout = st["inb"][slot], st["outb"][slot]
        with torch.cuda.stream(s_in):
            if c_done[slot] is not None:
                s_in.wait_event(c_done[slot])
            din[:k].copy_(x[f0:f0 + k], non_blocking=True)
            h_ev = torch.cuda.Event()
            h_ev.record(s_in)
        comp.wait_event(h_ev)
        if d_done[slot] is not None:
            comp.wait_event(d_done[slot])
        launch(k, din, dout, comp.cuda_stream)
        c_ev = torch.cuda.Event()
        c_ev.record(comp)
        c_done[slot] = c_ev
        with torch.cuda.stream(s_out):
            s_out.wait_event(c_ev)
            dst = out[f0:f0 + k] if finish is None else st["stage"][slot][:k]
            dst.copy_(dout[:k], non_blocking=True)
            d_ev = torch.cuda.Event()
            d_ev.record(s_out)
        d_done[slot] = d_ev
        if finish is not None:
            # the staging slot of chunk i-1 is reused by chunk i+1's copy,
            # which is only enqueued after this finish returns
            if pending is not None:
                pf0, pk, pslot, pev = pending
                pev.synchronize()
                finish(pf0, pk, st["stage"][pslot][:pk])
            pending = (f0, k, slot, d_ev)
    s_out.synchronize()
    if pending is not None:
        pf0, pk, pslot, _ = pending
        finish(pf0, pk, st["stage"][pslot][:pk])
    comp.wait_stream(s_out)
    return out


def edge_detection_pipelined(input, gaussian_filter, structure, sx, sy, theta, out=None, chunk: int = 16,
                             device=None, bits: bool = True):
    """Host-buffer edge detection with copy/compute overlap (``_pipelined``).

    ``input`` is a host f32[batch,n,m] (numpy or CPU torch tensor; pinned
    memory gives full PCIe bandwidth).  Returns ``out`` (a host f32 tensor of
    the input's shape).  ``bits`` (default) moves each chunk's maps
    device->host bit-packed (jb_edge_bits_f32) and expands them on the host
    (jb_bits_expand_f32): the same values, 1/32 of the D2H bytes."""
    torch = _torch()
    x = input if isinstance(input, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(input, np.float32))
    _need(x.dtype == torch.float32 and x.dim() == 3 and not x.is_cuda,
          "edge_detection_pipelined: input must be a host f32[batch,n,m]")
    B, n, m = (int(v) for v in x.shape)
    if out is None:
        out = torch.empty_like(x, pin_memory=x.is_pinned())
    gs, sz, sb = (_shape(f)[0] for f in (gaussian_filter, structure, sx))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    filt = [(f.to(dev) if isinstance(f, torch.Tensor) else
             torch.from_numpy(np.ascontiguousarray(f, np.float32)).to(dev))
            for f in (gaussian_filter, structure, sx, sy)]
    lib = _lib.load()

    if not bits:
        def launch(k, din, dout, stream):
            _check(lib.jb_edge_f32(k, n, m, gs, sz, sb, din.data_ptr(), filt[0].data_ptr(), filt[1].data_ptr(),
                                   filt[2].data_ptr(), filt[3].data_ptr(), _scalar(theta), dout.data_ptr(),
                                   stream), "edge_detection")
        with torch.cuda.device(dev):
            return _pipelined(x, out, chunk, "edge", launch, dev)

    # the edge map is exactly 0/1: it crosses PCIe as bits (1/32 of the f32
    # bytes) and is expanded into ``out`` on the host thread pool
    _need(out.dtype == torch.float32 and out.is_contiguous() and tuple(out.shape) == (B, n, m),
          "edge_detection_pipelined: out must be a contiguous host f32[batch,n,m]")
    fw = (n * m + 31) // 32
    out_ptr = out.data_ptr()

    def launch_bits(k, din, dout, stream):
        _check(lib.jb_edge_bits_f32(k, n, m, gs, sz, sb, din.data_ptr(), filt[0].data_ptr(),
                                    filt[1].data_ptr(), filt[2].data_ptr(), filt[3].data_ptr(), _scalar(theta),
                                    dout.data_ptr(), stream), "edge_detection")

    # 3 host threads: measured best on the B200 box (tools/e2e_probe2.py,
    # profiles/r02_e2e_probe.txt) -- the host's DRAM is shared by the DMA
    # reading the next chunk's input and this expansion writing the result,
    # and a full-pool expansion starves the DMA (55 -> 22-31 GB/s)
    def finish(f0, k, staged):
        _check(lib.jb_bits_expand_f32(staged.data_ptr(), k, n * m, out_ptr + f0 * n * m * 4, EXPAND_THREADS),
               "edge_detection (bit expansion)")
    with torch.cuda.device(dev):
        return _pipelined(x, out, chunk, "edge_bits", launch_bits, dev, out_elem=((fw,), torch.int32),
                          finish=finish)


def cava_pipelined(input, tstw, ctrl_pts, weights, coefs, tonemap, out=None, chunk: int = 8, device=None):
    """Host-buffer CAVA over a batch u8[batch,3,r,c] with copy/compute overlap
    (``_pipelined``); returns ``out`` (a host u8 tensor of the input's shape)."""
    torch = _torch()
    x = input if isinstance(input, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(input, np.uint8))
    _need(x.dtype == torch.uint8 and x.dim() == 4 and x.shape[1] == 3 and not x.is_cuda,
          "cava_pipelined: input must be a host u8[batch,3,r,c]")
    B, _, r, c = (int(v) for v in x.shape)
    if out is None:
        out = torch.empty_like(x, pin_memory=x.is_pinned())
    P = _shape(ctrl_pts)[0]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    prm = [(f.to(dev) if isinstance(f, torch.Tensor) else
            torch.from_numpy(np.ascontiguousarray(f, np.float32)).to(dev))
           for f in (tstw, ctrl_pts, weights, coefs, tonemap)]
    lib = _lib.load()

    def launch(k, din, dout, stream):
        _check(lib.jb_cava_u8(k, r, c, P, din.data_ptr(), *(t.data_ptr() for t in prm), dout.data_ptr(), stream),
               "cava")
    with torch.cuda.device(dev):
        return _pipelined(x, out, chunk, "cava", launch, dev)


def edge_detection_stages(input, gaussian_filter, structure, sx, sy, theta):
    """Stage-level variant (tests): returns dict of every intermediate."""
    shp = _shape(input)
    batch, n, m = (1, *shp) if len(shp) == 2 else shp
    gs, sz, sb = (_shape(x)[0] for x in (gaussian_filter, structure, sx))
    c = _Call([input, gaussian_filter, structure, sx, sy])
    din = c.dev(input, np.float32, "input")
    dg, dst, dsx, dsy = (c.dev(x, np.float32, "filter") for x in (gaussian_filter, structure, sx, sy))
    out, sm, lp, zc, gr = (c.empty(shp, np.float32) for _ in range(5))
    mx = c.empty((batch,), np.float32)
    with c.on_device():
        _check(_lib.load().jb_edge_stages_f32(batch, n, m, gs, sz, sb, _ptr(din), _ptr(dg), _ptr(dst),
                                              _ptr(dsx), _ptr(dsy), _scalar(theta), _ptr(out), _ptr(sm),
                                              _ptr(lp), _ptr(zc), _ptr(gr), _ptr(mx), c.s),
               "edge_detection_stages")
    return dict(out=c.out(out), smoothed=c.out(sm), laplacian=c.out(lp), zero_crossings=c.out(zc),
                gradient=c.out(gr), max_gradient=c.out(mx))


# ------------------------------------------------------------------------ cava
def cava(input, tstw, ctrl_pts, weights, coefs, tonemap):
    """cava<r,c,num_ctrl_pts>(input u8[3,r,c] | u8[batch,3,r,c], TsTw f32[3,3],
    ctrl_pts f32[P,3], weights f32[P,3], coefs f32[4,3], tonemap f32[256,3]) -> u8."""
    shp = _shape(input)
    _need(len(shp) in (3, 4) and shp[-3] == 3, "cava: input must be u8[3,r,c] or u8[batch,3,r,c]")
    batch = 1 if len(shp) == 3 else shp[0]
    r, cc = shp[-2], shp[-1]
    P = _shape(ctrl_pts)[0]
    _need(_shape(tstw) == (3, 3), "cava: TsTw must be f32[3,3]")
    _need(_shape(ctrl_pts) == (P, 3) and _shape(weights) == (P, 3), "cava: ctrl_pts/weights must be f32[P,3]")
    _need(_shape(coefs) == (4, 3), "cava: coefs must be f32[4,3]")
    _need(_shape(tonemap) == (256, 3), "cava: tonemap must be f32[256,3]")
    c = _Call([input, tstw, ctrl_pts, weights, coefs, tonemap])
    if c.host and len(shp) == 4 and batch > 1:
        x = hostmem.pinned_view(c.host_array(input, np.uint8, "input"))
        out = hostmem.pinned_empty(shp, _torch().uint8)
        cava_pipelined(x, tstw, ctrl_pts, weights, coefs, tonemap, out=out, device=c.device)
        return out.numpy()
    din = c.dev(input, np.uint8, "input")
    dt, dc, dw, dco, dtm = (c.dev(x, np.float32, nm) for x, nm in
                            ((tstw, "TsTw"), (ctrl_pts, "ctrl_pts"), (weights, "weights"),
                             (coefs, "coefs"), (tonemap, "tonemap")))
    out = c.empty(shp, np.uint8)
    with c.on_device():
        _check(_lib.load().jb_cava_u8(batch, r, cc, P, _ptr(din), _ptr(dt), _ptr(dc), _ptr(dw), _ptr(dco),
                                      _ptr(dtm), _ptr(out), c.s), "cava")
    return c.out(out)


# ------------------------------------------------------------------------ srad
def srad(niter, lam, image, return_q0sqr: bool = False, exact: bool = False):
    """srad<rows,cols>(niter, lambda, image f32[rows,cols]) -> f32[rows,cols].

    Default: tolerance mode (rel 1e-4 of the oracle after niter, DESIGN.md
    §srad).  ``exact=True``: the oracle's arithmetic op for op."""
    niter = _scalar(niter, int)
    if niter < 0:
        raise _err(DynConstError, f"srad: niter must be >= 0 (got {niter})")
    _need(len(_shape(image)) == 2, "srad: image must be f32[rows,cols]")
    rows, cols = _shape(image)
    c = _Call([image])
    dimg = c.dev(image, np.float32, "image")
    out = c.empty((rows, cols), np.float32)
    q0 = c.empty((max(niter, 1),), np.float32)
    with c.on_device():
        fn = _lib.load().jb_srad_exact_f32 if exact else _lib.load().jb_srad_f32
        _check(fn(rows, cols, niter, _scalar(lam), _ptr(dimg), _ptr(out), _ptr(q0), c.s), "srad")
    if return_q0sqr:
        return c.out(out), c.out(q0[:niter])
    return c.out(out)


# ----------------------------------------------------------------------- euler
def euler(iterations, areas, neighbors, normals, ff_variable, variables, exact: bool = False):
    """euler<nelr>(iterations, areas f32[nelr], neighbors i32[4,nelr],
    normals f32[4,3,nelr], ff_variable f32[5], variables f32[5,nelr]) -> f32[5,nelr].

    Default: tolerance mode (rel 1e-5 per RK stage).
    ``exact=True``: bit-identical to the oracle."""
    iterations = _scalar(iterations, int)
    if iterations < 0:
        raise _err(DynConstError, "euler: iterations must be >= 0")
    nelr = _shape(areas)[0]
    _need(_shape(neighbors) == (4, nelr), "euler: neighbors must be i32[4,nelr]")
    _need(_shape(normals) == (4, 3, nelr), "euler: normals must be f32[4,3,nelr]")
    _need(_shape(ff_variable) == (5,), "euler: ff_variable must be f32[5]")
    _need(_shape(variables) == (5, nelr), "euler: variables must be f32[5,nelr]")
    c = _Call([areas, neighbors, normals, ff_variable, variables])
    da = c.dev(areas, np.float32, "areas")
    dn = c.dev(neighbors, np.int32, "neighbors")
    dno = c.dev(normals, np.float32, "normals")
    dff = c.dev(ff_variable, np.float32, "ff_variable")
    dv = c.dev(variables, np.float32, "variables", copy=True)  # value semantics
    with c.on_device():
        fn = _lib.load().jb_euler_exact_f32 if exact else _lib.load().jb_euler_f32
        _check(fn(nelr, iterations, _ptr(da), _ptr(dn), _ptr(dno), _ptr(dff), _ptr(dv), c.s), "euler")
    return c.out(dv)


def euler_step_factor(variables, areas):
    nelr = _shape(areas)[0]
    c = _Call([variables, areas])
    dv, da = c.dev(variables, np.float32, "variables"), c.dev(areas, np.float32, "areas")
    out = c.empty((nelr,), np.float32)
    with c.on_device():
        _check(_lib.load().jb_euler_step_factor_f32(nelr, _ptr(dv), _ptr(da), _ptr(out), c.s), "euler_step_factor")
    return c.out(out)


def euler_flux(neighbors, normals, ff_variable, variables):
    nelr = _shape(neighbors)[1]
    c = _Call([neighbors, normals, ff_variable, variables])
    dn = c.dev(neighbors, np.int32, "neighbors")
    dno, dff, dv = (c.dev(x, np.float32, "f") for x in (normals, ff_variable, variables))
    out = c.empty((5, nelr), np.float32)
    with c.on_device():
        _check(_lib.load().jb_euler_flux_f32(nelr, _ptr(dn), _ptr(dno), _ptr(dff), _ptr(dv), _ptr(out), c.s),
               "euler_flux")
    return c.out(out)


# ------------------------------------------------------------------------- bfs
def bfs(starting, no_of_edges, edges, source):
    """bfs<n,m>(starting u32[n], no_of_edges u32[n], edges u32[m], source) -> i32[n]."""
    n = _shape(starting)[0]
    m = _shape(edges)[0]
    _need(_shape(no_of_edges) == (n,), "bfs: no_of_edges must be u32[n]")
    source = _scalar(source, int)
    _need(n == 0 or 0 <= source < n, f"bfs: source {source} out of bounds for n={n}")
    c = _Call([starting, no_of_edges, edges])
    ds = c.dev(starting, np.uint32, "starting")
    dne = c.dev(no_of_edges, np.uint32, "no_of_edges")
    de = c.dev(edges, np.uint32, "edges") if m else c.empty((1,), np.int32)
    cost = c.empty((n,), np.int32)
    with c.on_device():
        _check(_lib.load().jb_bfs(n, m, _ptr(ds), _ptr(dne), _ptr(de), source, _ptr(cost), c.s), "bfs")
    return c.out(cost)


# -------------------------------------------------------------------- backprop
def backprop(input_vals, input_weights, hidden_weights, target, input_prev_weights, hidden_prev_weights,
             return_layers: bool = False):
    """One Rodinia bpnn_train step (layerforward x2, output/hidden error,
    adjust_weights x2).  Returns (out_err, hid_err, input_weights,
    hidden_weights, input_prev_weights, hidden_prev_weights) -- fresh arrays
    (value semantics; the inputs are not mutated) -- plus (hidden, output)
    unit values when ``return_layers``."""
    n_in1, n_hid1 = _shape(input_weights)
    n_hid1b, n_out1 = _shape(hidden_weights)
    _need(n_hid1 == n_hid1b, "backprop: weight shapes disagree on the hidden layer")
    _need(_shape(input_vals) == (n_in1,), "backprop: input_vals must be f32[n_in+1]")
    _need(_shape(target) == (n_out1,), "backprop: target must be f32[n_out+1]")
    _need(_shape(input_prev_weights) == (n_in1, n_hid1), "backprop: input_prev_weights shape")
    _need(_shape(hidden_prev_weights) == (n_hid1, n_out1), "backprop: hidden_prev_weights shape")
    c = _Call([input_vals, input_weights, hidden_weights, target, input_prev_weights, hidden_prev_weights])
    dx = c.dev(input_vals, np.float32, "input_vals", copy=True)
    diw = c.dev(input_weights, np.float32, "input_weights", copy=True)
    dhw = c.dev(hidden_weights, np.float32, "hidden_weights", copy=True)
    dt = c.dev(target, np.float32, "target")
    dipw = c.dev(input_prev_weights, np.float32, "input_prev_weights", copy=True)
    dhpw = c.dev(hidden_prev_weights, np.float32, "hidden_prev_weights", copy=True)
    hidden = c.empty((n_hid1,), np.float32)
    output = c.empty((n_out1,), np.float32)
    errs = c.empty((2,), np.float32)
    with c.on_device():
        _check(_lib.load().jb_bp_train_f32(n_in1 - 1, n_hid1 - 1, n_out1 - 1, _ptr(dx), _ptr(diw), _ptr(dhw),
                                           _ptr(dt), _ptr(dipw), _ptr(dhpw), _ptr(hidden), _ptr(output),
                                           _ptr(errs), c.s), "backprop")
    e = c.out(errs)
    res = (e[0], e[1], c.out(diw), c.out(dhw), c.out(dipw), c.out(dhpw))
    return res + (c.out(hidden), c.out(output)) if return_layers else res


# --------------------------------------------------------- oracle_execute mirror
@dataclass(frozen=True)
class Entry:
    dyn_consts: tuple[str, ...]
    shapes: Callable[[Sequence[int], Sequence[Any]], list]  # expected (arg idx, shape) pairs
    run: Callable[..., Any]
    # device memory the entry function takes for its results and working
    # copies, as (shape, dtype) in request order, from the dyn-consts and
    # arguments alone: the runner's allocation plan (runner.py)
    results: Callable[[Sequence[int], Sequence[Any]], list] = lambda d, a: []


def _sh(*pairs):
    return list(pairs)


ENTRIES: dict[str, Entry] = {
    "matmul": Entry(("n", "m", "l"),
                    lambda d, a: _sh((0, (d[0], d[1])), (1, (d[1], d[2]))),
                    lambda d, a, **kw: matmul(*a, **kw),
                    lambda d, a: [((d[0], d[2]), np.float32)]),
    "edge_detection": Entry(("n", "m", "gs", "sz", "sb"),
                            lambda d, a: _sh((0, (d[0], d[1])), (1, (d[2], d[2])), (2, (d[3], d[3])),
                                             (3, (d[4], d[4])), (4, (d[4], d[4]))),
                            lambda d, a: edge_detection(*a),
                            lambda d, a: [(_shape(a[0]), np.float32)]),
    "cava": Entry(("r", "c", "num_ctrl_pts"),
                  lambda d, a: _sh((0, (3, d[0], d[1])), (1, (3, 3)), (2, (d[2], 3)), (3, (d[2], 3)),
                                   (4, (4, 3)), (5, (256, 3))),
                  lambda d, a: cava(*a),
                  lambda d, a: [(_shape(a[0]), np.uint8)]),
    "srad": Entry(("nrows", "ncols"),
                  lambda d, a: _sh((2, (d[0], d[1]))),
                  lambda d, a: srad(*a),
                  lambda d, a: [((d[0], d[1]), np.float32), ((max(int(a[0]), 1),), np.float32)]),
    "euler": Entry(("nelr",),
                   lambda d, a: _sh((1, (d[0],)), (2, (4, d[0])), (3, (4, 3, d[0])), (4, (5,)), (5, (5, d[0]))),
                   lambda d, a: euler(*a),
                   lambda d, a: [((5, d[0]), np.float32)]),
    "bfs": Entry(("n", "m"),
                 lambda d, a: _sh((0, (d[0],)), (1, (d[0],)), (2, (d[1],))),
                 lambda d, a: bfs(*a),
                 lambda d, a: ([((1,), np.int32)] if d[1] == 0 else []) + [((d[0],), np.int32)]),
    "backprop": Entry(("input_n", "hidden_n", "output_n"),
                      lambda d, a: _sh((0, (d[0] + 1,)), (1, (d[0] + 1, d[1] + 1)), (2, (d[1] + 1, d[2] + 1)),
                                       (3, (d[2] + 1,)), (4, (d[0] + 1, d[1] + 1)), (5, (d[1] + 1, d[2] + 1))),
                      lambda d, a: backprop(*a),
                      lambda d, a: [((d[0] + 1,), np.float32), ((d[0] + 1, d[1] + 1), np.float32),
                                    ((d[1] + 1, d[2] + 1), np.float32), ((d[0] + 1, d[1] + 1), np.float32),
                                    ((d[1] + 1, d[2] + 1), np.float32), ((d[1] + 1,), np.float32),
                                    ((d[2] + 1,), np.float32), ((2,), np.float32)]),
}


def execute(entry: str, dyn_consts, args, params: Optional[dict] = None):
    """Run Juno ``entry`` on the B200: ``oracle_execute`` without the module
    (the entry names the benchmark program of SURVEY.md §8 (a.2)).
    ``params``: launch parameters a schedule implies (planner.select_kernel;
    matmul: ``tile_n``, ``tree``)."""
    dcs, args = validate(entry, dyn_consts, args)
    if params:
        return ENTRIES[entry].run(dcs, args, **params)
    return ENTRIES[entry].run(dcs, args)


# argument index that may carry a leading batch dimension (independent frames)
BATCHED_ARG = {"edge_detection": 0, "cava": 0}


def validate(entry: str, dyn_consts, args):
    """The invocation checks of ``execute``: entry known, dynamic constants
    counted and non-negative (dynconst.py:179-204), argument extents equal to
    the ones the dynamic constants give (edge/cava input may add a leading
    batch dimension).  Returns (dcs, args)."""
    if entry not in ENTRIES:
        raise _err(RuntimeError_, f"no B200 kernel for entry {entry!r}; known: {sorted(ENTRIES)}")
    spec = ENTRIES[entry]
    dcs = [int(x) for x in dyn_consts]
    if len(dcs) != len(spec.dyn_consts):
        raise _err(DynConstError, f"{entry}: expected {len(spec.dyn_consts)} dynamic constants "
                                  f"{spec.dyn_consts}, got {len(dcs)}")
    for nm, v in zip(spec.dyn_consts, dcs):
        if v < 0:
            raise _err(DynConstError, f"{entry}: dynamic constant {nm} = {v} is negative")
    args = list(args)
    for idx, want in spec.shapes(dcs, args):
        if idx >= len(args):
            raise _err(RuntimeError_, f"{entry}: missing argument {idx}")
        got, want = _shape(args[idx]), tuple(want)
        batched = BATCHED_ARG.get(entry) == idx and len(got) == len(want) + 1 and got[1:] == want
        if got != want and not batched:
            raise _err(RuntimeError_, f"{entry}: argument {idx} has shape {got}, expected {want} "
                                      f"under dyn-consts {dict(zip(spec.dyn_consts, dcs))}")
    return dcs, args


def _raise_dc(msg, cause):
    raise _err(DynConstError, msg) from cause


def oracle_execute(module, entry: str, dyn_consts, args, max_steps: int = 50_000_000):
    """Drop-in for skiff.runtime.oracle.oracle_execute (oracle.py:28-32).

    ``module`` is a skiff ``Module``.  Its function ``entry`` (KeyError when
    absent, as oracle.py:30) is first held to its invocation contract --
    divisibility constraints and exact dynamic-constant evaluation, raising
    ``DynConstError`` as the reference does (recognize.check_invocation) --
    then recognised structurally (recognize.recognize: the body, not the name
    or signature).  A function no kernel computes raises
    ``UnsupportedError``.  ``module=None`` runs the benchmark program named
    by ``entry`` directly (``execute``).  ``max_steps`` is accepted for
    signature parity; the device path has no interpreter budget."""
    del max_steps
    if module is None:
        return execute(entry, dyn_consts, args)
    fns = getattr(module, "functions", None)
    if fns is None:
        raise _err(RuntimeError_, f"oracle_execute: {type(module).__name__} is not a Module")
    fn = fns[entry]
    from .recognize import check_invocation, recognize
    dcs = check_invocation(fn, dyn_consts, _raise_dc)
    args = list(args)
    if len(args) != len(fn.param_types):
        raise _err(RuntimeError_, f"{entry}: expected {len(fn.param_types)} arguments, got {len(args)}")
    rec, why = recognize(fn, dcs)
    if rec is None:
        raise _err(UnsupportedError, f"no B200 kernel computes function {entry!r}: " +
                   "; ".join(f"not {k} ({v})" for k, v in why.items()))
    return execute(rec.entry, rec.dyn_consts, args, rec.params)
