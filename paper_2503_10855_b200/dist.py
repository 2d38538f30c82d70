"""Multi-GPU partitioning of the Juno benchmarks.

One process per GPU (torch.distributed; NCCL over NVLink on the B200 box,
gloo in the CPU tests).  What shards and how:

  edge, CAVA   frames split across ranks, no collective      (shard_frames)
  matmul       row blocks of A and C, B replicated once       (row_block, matmul_row_blocks)
  SRAD         row slabs with 1 halo row above / 2 below; per iteration an
               allreduce of the f64 (sum, sum^2) pair and a halo exchange of
               the image rows                                 (srad_distributed)
  CFD/Euler    contiguous element ranges; the halo is every element an owned
               element's neighbour list points outside the range (one mesh row
               above and below on the structured mesh); per RK stage a halo
               exchange of the 5 variables              (euler_plan, euler_distributed)
  BFS, BP      replicas only

The SRAD driver is written against a small backend protocol so the same host
logic runs on the GPU (``CudaSradBackend``: libjunob200 slab kernels, device
tensors, NCCL) and in the gloo tests (a CPU backend the tests provide).  The
result is bit-identical to the single-device run whenever the allreduced f64
sums round to the same f32 q0^2 as the single-device sums.
"""

from __future__ import annotations

from typing import Protocol

from . import _lib


def partition(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of n units: (first, count) of `rank`."""
    base, extra = divmod(int(n), int(world))
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def shard_frames(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Frames of a batched edge/CAVA call owned by `rank` (no collective)."""
    return partition(batch, world, rank)


def row_block(n: int, world: int, rank: int) -> tuple[int, int]:
    """Rows of A and C owned by `rank` for a row-block matmul."""
    return partition(n, world, rank)


class MatmulRowBlocks:
    """Row-block matmul<n,m,l> across the ranks of `group`.

    A and C are split by rows (row_block); B is replicated: it is broadcast
    from `src` ONCE, when the object is built, and cached on every rank, so a
    call is collective-free -- each rank runs the tcgen05 kernel on its own
    rows (`mm`, default api.matmul; the CPU tests pass the oracle).
    ``gather(c_rows)`` all-gathers the full C when one rank needs it."""

    def __init__(self, b, n: int, group=None, src: int = 0, mm=None):
        import torch.distributed as dist
        self.group, self.n = group, int(n)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.r0, self.rows = row_block(self.n, self.world, self.rank)
        if self.world > 1:
            b = b.contiguous()
            if b.is_cuda and _gloo(group):   # shared-GPU test mode: stage through the host
                x = b.cpu()
                dist.broadcast(x, src=src, group=group)
                b.copy_(x)
            else:
                dist.broadcast(b, src=src, group=group)
        self.b = b
        if mm is None:
            from .api import matmul as mm
        self.mm = mm
        self.broadcasts = 1 if self.world > 1 else 0

    def own_rows(self, a_full):
        """This rank's rows of a full A."""
        return a_full[self.r0:self.r0 + self.rows]

    def __call__(self, a_rows):
        assert a_rows.shape[0] == self.rows, f"rank {self.rank} owns {self.rows} rows, got {a_rows.shape[0]}"
        return self.mm(a_rows, self.b)

    def gather(self, c_rows):
        """The full C on every rank (all-gather of the row blocks)."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return c_rows
        t = c_rows if isinstance(c_rows, torch.Tensor) else torch.from_numpy(c_rows)
        cap = -(-self.n // self.world)
        pad = torch.zeros((cap, t.shape[1]), dtype=t.dtype, device=t.device)
        pad[:self.rows] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        if pad.is_cuda and _gloo(self.group):
            cpu = [p.cpu() for p in parts]
            dist.all_gather(cpu, pad.cpu(), group=self.group)
            parts = [c.to(pad.device) for c in cpu]
        else:
            dist.all_gather(parts, pad, group=self.group)
        full = torch.cat([p[:row_block(self.n, self.world, r)[1]] for r, p in enumerate(parts)])
        return full if isinstance(c_rows, torch.Tensor) else full.numpy()


def matmul_row_blocks(a_rows, b, n: int = None, group=None, src: int = 0):
    """One-shot row-block matmul: C[rows] = A[rows] @ B with B broadcast from
    `src` (for repeated calls build a MatmulRowBlocks: it broadcasts once)."""
    n = a_rows.shape[0] if n is None else n
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mb = MatmulRowBlocks(b, n if world > 1 else a_rows.shape[0], group, src)
    return mb(a_rows)


# ------------------------------------------------------------------- SRAD
def srad_slab(rows: int, world: int, rank: int) -> dict:
    """Owned rows [r0, r1) and the extended slab [e0, e1) with the halos the
    fused kernel needs (north 1 row, south 2 rows: the coefficient of the
    first row below the slab is recomputed locally)."""
    if rows < 2 * world:
        raise ValueError(f"srad_distributed needs >= 2 rows per rank ({rows} rows, {world} ranks)")
    r0, cnt = partition(rows, world, rank)
    r1 = r0 + cnt
    e0, e1 = max(r0 - 1, 0), min(r1 + 2, rows)
    return dict(r0=r0, r1=r1, e0=e0, e1=e1, own_lo=r0 - e0, own_hi=r1 - e0)


class SradBackend(Protocol):
    def extract(self, image_own, compress: bool): ...            # -> (J_own, sums f64[2])
    def step(self, J_ext, own_lo: int, own_hi: int, q0, lam: float, compress: bool, out=None): ...
    # -> (out_own, sums); writes into `out` (own rows of the other slab buffer) when given
    def q0(self, sums, npx: int): ...                              # -> q0 (backend tensor)
    def empty_rows(self, n: int, cols: int, like): ...             # -> uninitialised [n, cols]
    def cat_rows(self, parts): ...


def _gloo(group) -> bool:
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _p2p(ops_spec, group):
    """Batched isend/irecv of (kind, tensor, peer) triples.  NCCL moves the
    device tensors directly; a gloo group (CPU tests, the shared-GPU bench
    test mode) stages CUDA tensors through host copies."""
    import torch.distributed as dist
    staged, ops = [], []
    for kind, t, peer in ops_spec:
        x = t
        if t.is_cuda and _gloo(group):
            x = t.detach().cpu() if kind == "send" else torch_empty_cpu(t)
            staged.append((kind, t, x))
        ops.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, x.contiguous() if kind == "send" else x,
                              peer, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for kind, t, x in staged:
        if kind == "recv":
            t.copy_(x)


def torch_empty_cpu(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype)


def _all_reduce(t, group):
    import torch.distributed as dist
    if t.is_cuda and _gloo(group):
        x = t.cpu()
        dist.all_reduce(x, group=group)
        t.copy_(x)
    else:
        dist.all_reduce(t, group=group)


def _halo_exchange_rows(ext, lo: int, hi: int, rank: int, world: int, group):
    """In place: ext = [north 1 | own rows lo..hi | south 2] of this rank's
    slab (rows that exist); the halo rows are received straight into it."""
    spec = []
    if rank > 0:
        spec.append(("recv", ext[0:1], rank - 1))
        spec.append(("send", ext[lo:lo + 2], rank - 1))
    if rank < world - 1:
        spec.append(("recv", ext[hi:hi + 2], rank + 1))
        spec.append(("send", ext[hi - 1:hi], rank + 1))
    _p2p(spec, group)


def srad_distributed(image_own, niter: int, lam: float, rows: int, cols: int, backend: SradBackend,
                     group=None):
    """Row-slab SRAD across the ranks of `group`.  `image_own` holds this
    rank's rows (srad_slab(...)[r0:r1]); returns this rank's output rows.
    Two extended slab buffers [north 1 | own | south 2] are reused: the step
    kernel writes the new own rows into the other buffer and the halo rows
    are received in place (no per-iteration slab copy)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    plan = srad_slab(rows, world, rank)
    assert image_own.shape[0] == plan["r1"] - plan["r0"] and image_own.shape[1] == cols
    npx = rows * cols
    if niter == 0:
        out, _ = backend.extract(image_own, compress=True)
        return out
    lo, hi, n_ext = plan["own_lo"], plan["own_hi"], plan["e1"] - plan["e0"]
    J, sums = backend.extract(image_own, compress=False)
    ext = [backend.empty_rows(n_ext, cols, like=J) for _ in range(2)]
    ext[0][lo:hi] = J
    if world > 1:
        _all_reduce(sums, group)
    q0 = backend.q0(sums, npx)
    cur = 0
    for it in range(niter):
        last = it + 1 == niter
        if world > 1:
            _halo_exchange_rows(ext[cur], lo, hi, rank, world, group)
        _, sums = backend.step(ext[cur], lo, hi, q0, lam, compress=last, out=ext[cur ^ 1][lo:hi])
        cur ^= 1
        if not last:
            if world > 1:
                _all_reduce(sums, group)
            q0 = backend.q0(sums, npx)
    return ext[cur][lo:hi]


class _Raw:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3}


def _raw_tensor(ptr: int, shape, dtype="f4"):
    import torch
    return torch.as_tensor(_Raw(ptr, shape, "<" + dtype), device="cuda")


class SradP2PSlabs:
    """Peer-memory slab buffers of one rank for the fused multi-GPU SRAD step.

    One IPC-exportable allocation per rank holds [ext 0 | ext 1 | mailbox |
    counter]: two extended slabs [north 1 | own | south 2] and the mailbox the
    other ranks write their (sum, sum^2) into.  The handles are exchanged once
    (all_gather_object) and every peer allocation is mapped
    (cudaIpcOpenMemHandle: NVLink P2P between GPUs; the same device in the
    one-GPU tests)."""

    MBOX = 256  # bytes: double[2][8][2]

    def __init__(self, rows: int, cols: int, group=None, grid: int = 0):
        import ctypes
        import torch.distributed as dist
        self.lib = _lib.load()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > 8:
            raise ValueError("the fused P2P step supports up to 8 ranks")
        if cols % 4:
            raise ValueError("the fused P2P step needs cols % 4 == 0")
        self.rows, self.cols, self.group, self.grid = rows, cols, group, grid
        self.epoch = 0  # this rank's arrival counter after the calls so far
        self.plans = [srad_slab(rows, self.world, r) for r in range(self.world)]
        self.ext_bytes = [(p["e1"] - p["e0"]) * cols * 4 for p in self.plans]
        nbytes = 2 * self.ext_bytes[self.rank] + self.MBOX + 256
        ptr = ctypes.c_void_p()
        self._chk(self.lib.jb_p2p_alloc(nbytes, ctypes.byref(ptr)), "p2p_alloc")
        self.base = ptr.value
        h = ctypes.create_string_buffer(64)
        self._chk(self.lib.jb_ipc_handle(self.base, h), "ipc_handle")
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, h.raw, group=group)
        else:
            handles = [h.raw]
        self.peers, self.opened = [], []
        for r in range(self.world):
            if r == self.rank:
                self.peers.append(self.base)
                continue
            p = ctypes.c_void_p()
            self._chk(self.lib.jb_ipc_open(ctypes.create_string_buffer(handles[r], 64), ctypes.byref(p)),
                      f"ipc_open(rank {r})")
            self.peers.append(p.value)
            self.opened.append(p.value)

    def _chk(self, rc, what):
        if rc:
            raise RuntimeError(f"{what}: {_lib.last_error()}")

    def ext(self, b: int, r: int = None) -> int:  # device address of slab buffer b of rank r
        r = self.rank if r is None else r
        return self.peers[r] + b * self.ext_bytes[r]

    def mbox(self, r: int) -> int:
        return self.peers[r] + 2 * self.ext_bytes[r]

    def flag(self, r: int) -> int:
        return self.mbox(r) + self.MBOX

    def ext_tensor(self, b: int):
        p = self.plans[self.rank]
        return _raw_tensor(self.ext(b), (p["e1"] - p["e0"], self.cols))

    def close(self):
        for p in self.opened:
            self.lib.jb_ipc_close(p)
        self.opened = []
        if self.base:
            self.lib.jb_p2p_free(self.base)
            self.base = None


def srad_distributed_p2p(image_own, niter: int, lam: float, slabs: SradP2PSlabs, backend=None,
                         exact: bool = False):
    """Row-slab SRAD where each iteration is ONE kernel per rank: it stores
    the slab's boundary rows into the neighbours' next slabs and its sums into
    every rank's mailbox over peer memory, and the next iteration's kernel
    waits on the arrival counter (jb_srad_slab_p2p_step_f32).  The extract
    prologue runs once through the collective path.  Returns this rank's
    output rows (a copy)."""
    import ctypes
    import torch
    import torch.distributed as dist
    be = backend or CudaSradBackend()
    lib, w, rank, group = slabs.lib, slabs.world, slabs.rank, slabs.group
    plan = slabs.plans[rank]
    lo, hi, cols = plan["own_lo"], plan["own_hi"], slabs.cols
    npx = slabs.rows * cols
    if niter == 0:
        out, _ = be.extract(image_own, compress=True)
        return out
    # no host synchronisation between calls: the counters only grow (every
    # iteration adds `world` on every rank), so this call's iteration 0 waits
    # for the previous call to have finished everywhere (flag_base)
    ext0 = slabs.ext_tensor(0)
    J, sums = be.extract(image_own, compress=False)
    ext0[lo:hi] = J
    if w > 1:
        _all_reduce(sums, group)
        _halo_exchange_rows(ext0, lo, hi, rank, w, group)
    q0 = be.q0(sums, npx)
    a = _lib.SradP2P()
    a.mbox, a.flag = slabs.mbox(rank), slabs.flag(rank)
    for r in range(w):
        a.peer_mbox[r] = slabs.mbox(r)
        a.peer_flag[r] = slabs.flag(r)
    a.world, a.rank, a.npx_global, a.grid = w, rank, npx, slabs.grid
    a.flag_base = slabs.epoch
    stream = torch.cuda.current_stream().cuda_stream
    n_ext = plan["e1"] - plan["e0"]
    for it in range(niter):
        cur, nxt = it & 1, (it & 1) ^ 1
        last = it + 1 == niter
        a.iter = it
        a.peer_north = (slabs.ext(nxt, rank - 1) + slabs.plans[rank - 1]["own_hi"] * cols * 4) if rank > 0 else None
        a.peer_south = slabs.ext(nxt, rank + 1) if rank < w - 1 else None
        rc = lib.jb_srad_slab_p2p_step_f32(n_ext, cols, lo, hi, slabs.ext(cur), slabs.ext(nxt) + lo * cols * 4,
                                            q0.data_ptr() if it == 0 else None, float(lam), int(last),
                                            int(exact), ctypes.byref(a), stream)
        if rc:
            raise RuntimeError(f"srad_p2p_step: {_lib.last_error()}")
    slabs.epoch += w * niter
    return slabs.ext_tensor(niter & 1)[lo:hi].clone()


class CudaSradBackend:
    """libjunob200 slab kernels on device tensors (NCCL collectives).
    exact=True: the bit-exact slab step (else the tolerance mode of
    jb_srad_f32)."""

    def __init__(self, exact: bool = False):
        import torch
        self.torch = torch
        self.lib = _lib.load()
        self.exact = exact

    def _s(self):
        return self.torch.cuda.current_stream().cuda_stream

    def _chk(self, rc, what):
        if rc:
            raise RuntimeError(f"{what}: {_lib.last_error()}")

    def extract(self, image_own, compress):
        t = self.torch
        out = t.empty_like(image_own)
        sums = t.zeros(2, dtype=t.float64, device=image_own.device)
        self._chk(self.lib.jb_srad_extract_f32(image_own.numel(), image_own.data_ptr(), out.data_ptr(),
                                               None if compress else sums.data_ptr(), int(compress),
                                               self._s()), "srad_extract")
        return out, sums

    def empty_rows(self, n, cols, like):
        return self.torch.empty((n, cols), dtype=self.torch.float32, device=like.device)

    def step(self, J_ext, own_lo, own_hi, q0, lam, compress, out=None):
        t = self.torch
        if out is None:
            out = t.empty((own_hi - own_lo, J_ext.shape[1]), dtype=t.float32, device=J_ext.device)
        sums = t.zeros(2, dtype=t.float64, device=J_ext.device)
        self._chk(self.lib.jb_srad_slab_step_f32(J_ext.shape[0], J_ext.shape[1], own_lo, own_hi,
                                                 J_ext.data_ptr(), out.data_ptr(), q0.data_ptr(), float(lam),
                                                 sums.data_ptr(), int(compress), int(self.exact), self._s()),
                  "srad_slab_step")
        return out, sums

    def q0(self, sums, npx):
        q = self.torch.empty(1, dtype=self.torch.float32, device=sums.device)
        self._chk(self.lib.jb_srad_q0_f32(sums.data_ptr(), int(npx), q.data_ptr(), self._s()), "srad_q0")
        return q

    def cat_rows(self, parts):
        return self.torch.cat(parts, dim=0).contiguous()


# ------------------------------------------------------------------- CFD
def euler_plan(neighbors, world: int, rank: int) -> dict:
    """Element-range slab of `rank` for euler<nelr> and its halo exchange.

    `neighbors` is the global i32[4, nelr] array (ids, -1 wall, -2 far field).
    Returns the owned range [e0, e1), the slab-local neighbour ids (own
    elements 0..n_own-1, then the halo elements in global order), and per peer
    rank the own elements to send and the halo positions to receive.  Computed
    once per mesh on the host (numpy)."""
    import numpy as np
    nb = np.asarray(neighbors)
    nelr = nb.shape[1]
    bounds = [partition(nelr, world, r) for r in range(world)]

    def halo_of(r):
        e0, cnt = bounds[r]
        own = nb[:, e0:e0 + cnt]
        ext = own[(own >= 0) & ((own < e0) | (own >= e0 + cnt))]
        return np.unique(ext)

    e0, n_own = bounds[rank]
    e1 = e0 + n_own
    halo = halo_of(rank)
    own = nb[:, e0:e1]
    loc = own.astype(np.int64).copy()
    inside = (own >= e0) & (own < e1)
    outside = (own >= 0) & ~inside
    loc[inside] -= e0
    loc[outside] = n_own + np.searchsorted(halo, own[outside])
    starts = np.array([b[0] for b in bounds] + [nelr])
    owner = np.searchsorted(starts, halo, side="right") - 1
    recv = {}
    for r in np.unique(owner):
        pos = np.nonzero(owner == r)[0]
        recv[int(r)] = (int(pos[0]), int(pos.size))  # contiguous: halo is sorted by global id
    send = {}
    for s in range(world):
        if s == rank:
            continue
        h = halo_of(s)
        mine = h[(h >= e0) & (h < e1)]
        if mine.size:
            send[s] = (mine - e0).astype(np.int64)
    return dict(e0=e0, e1=e1, n_own=n_own, n_loc=n_own + halo.size, halo=halo,
                neighbors=np.ascontiguousarray(loc.astype(np.int32)), recv=recv, send=send)


def euler_plans(neighbors, world: int) -> list:
    """euler_plan for every rank (each rank's halo computed once)."""
    return [euler_plan(neighbors, world, r) for r in range(world)]


def euler_halo_exchange(cur, plan: dict, group=None, backend=None):
    """Fill the halo columns of the SoA slab array cur[5, n_loc] from their
    owners (batched point-to-point send/recv of the owned values they need)."""
    import torch
    n_own = plan["n_own"]
    spec, rbufs = [], []
    cache = plan.setdefault("_send_ids", {})  # device copies of the send lists, made once
    for s, idx in plan["send"].items():
        ids = cache.get((s, str(cur.device)))
        if ids is None:
            ids = cache[(s, str(cur.device))] = torch.as_tensor(idx, device=cur.device)
        spec.append(("send", cur.index_select(1, ids), s))
    for r, (st, cnt) in plan["recv"].items():
        buf = torch.empty((cur.shape[0], cnt), dtype=cur.dtype, device=cur.device)
        spec.append(("recv", buf, r))
        rbufs.append((st, cnt, buf))
    _p2p(spec, group)
    for st, cnt, buf in rbufs:
        cur[:, n_own + st:n_own + st + cnt] = buf


def euler_distributed(plan: dict, areas_own, normals_own, ff, vars_loc, iterations: int, backend,
                      group=None, exchange=None):
    """Rodinia euler on the slab of `plan`: `vars_loc` is the SoA f32[5, n_loc]
    slab state (own columns first; halo columns are filled here), updated in
    place; returns its own columns.  Per iteration the three RK stages each
    start with a halo exchange of the stage input (no reductions: the
    result is bit-identical to the single-device run)."""
    import torch
    exchange = exchange or (lambda cur: euler_halo_exchange(cur, plan, group))
    key = ("_nbrs", str(getattr(vars_loc, "device", "cpu")))
    if key not in plan:  # the slab-local neighbour ids move to the device once
        plan[key] = backend.to_device(plan["neighbors"], like=vars_loc)
    nbrs = plan[key]
    t1, t2 = torch.empty_like(vars_loc), torch.empty_like(vars_loc)
    for _ in range(iterations):
        for j, (cur, dst) in enumerate(((vars_loc, t1), (t1, t2), (t2, vars_loc))):
            exchange(cur)
            backend.stage(plan["n_own"], plan["n_loc"], j, areas_own, nbrs, normals_own, ff, cur, vars_loc, dst)
    return vars_loc[:, :plan["n_own"]]


class EulerP2PSlabs:
    """Peer-memory slab arrays of one rank for the fused multi-GPU CFD step.

    One IPC-exportable allocation per rank holds the three SoA stage arrays
    [V | t1 | t2] ([5][n_loc] each: own columns, then halo columns) and an
    arrival counter.  After each stage a push kernel stores the values the
    peers need straight into the peers' array of the same role and counts one
    arrival on each of them; the next stage waits on its own counter."""

    def __init__(self, neighbors, group=None, plans=None):
        import ctypes
        import numpy as np
        import torch
        import torch.distributed as dist
        self.lib = _lib.load()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > 8:
            raise ValueError("the fused P2P step supports up to 8 ranks")
        self.group = group
        self.plans = plans or euler_plans(neighbors, self.world)
        me = self.plan = self.plans[self.rank]
        self.arr_bytes = [5 * p["n_loc"] * 4 for p in self.plans]
        ptr = ctypes.c_void_p()
        self._chk(self.lib.jb_p2p_alloc(3 * self.arr_bytes[self.rank] + 256, ctypes.byref(ptr)), "p2p_alloc")
        self.base = ptr.value
        h = ctypes.create_string_buffer(64)
        self._chk(self.lib.jb_ipc_handle(self.base, h), "ipc_handle")
        handles = [h.raw]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, h.raw, group=group)
        self.peers, self.opened = [], []
        for r in range(self.world):
            if r == self.rank:
                self.peers.append(self.base)
                continue
            p = ctypes.c_void_p()
            self._chk(self.lib.jb_ipc_open(ctypes.create_string_buffer(handles[r], 64), ctypes.byref(p)),
                      f"ipc_open(rank {r})")
            self.peers.append(p.value)
            self.opened.append(p.value)
        # push list: (own element, destination rank, column in its arrays)
        own, peer, col = [], [], []
        for s, idx in me["send"].items():
            ps = self.plans[s]
            own.append(idx)
            peer.append(np.full(idx.size, s))
            col.append(ps["n_own"] + np.searchsorted(ps["halo"], me["e0"] + idx))
        dev = torch.device("cuda", torch.cuda.current_device())
        cat = (lambda xs: np.concatenate(xs).astype(np.int32)) if own else (lambda xs: np.zeros(0, np.int32))
        self.push_own = torch.from_numpy(cat(own)).to(dev)
        self.push_peer = torch.from_numpy(cat(peer)).to(dev)
        self.push_col = torch.from_numpy(cat(col)).to(dev)
        self.receivers = sorted(me["send"])
        self.srcmask = sum(1 << r for r in me["recv"])  # ranks that push into this one
        self.epoch = 0

    def _chk(self, rc, what):
        if rc:
            raise RuntimeError(f"{what}: {_lib.last_error()}")

    def buf(self, b: int, r: int = None) -> int:  # array b (0: V, 1: t1, 2: t2) of rank r
        r = self.rank if r is None else r
        return self.peers[r] + b * self.arr_bytes[r]

    def flags(self, r: int = None) -> int:  # rank r's counters, one u32 per source rank
        r = self.rank if r is None else r
        return self.peers[r] + 3 * self.arr_bytes[r]

    def array(self, b: int):
        return _raw_tensor(self.buf(b), (5, self.plan["n_loc"]))

    def push(self, b: int, stream):
        import ctypes
        w = self.world
        bufs = (ctypes.c_void_p * 8)(*[self.buf(b, r) for r in range(w)])
        strides = (ctypes.c_uint64 * 8)(*[p["n_loc"] for p in self.plans])
        flags = (ctypes.c_void_p * 8)(*[self.flags(r) + 4 * self.rank for r in self.receivers])
        self._chk(self.lib.jb_euler_push_f32(self.buf(b), self.plan["n_loc"], self.push_own.data_ptr(),
                                             self.push_peer.data_ptr(), self.push_col.data_ptr(),
                                             self.push_own.numel(), bufs, strides, flags, len(self.receivers),
                                             w, stream), "euler_push")

    def close(self):
        for p in self.opened:
            self.lib.jb_ipc_close(p)
        self.opened = []
        if self.base:
            self.lib.jb_p2p_free(self.base)
            self.base = None


def euler_distributed_p2p(slabs: EulerP2PSlabs, areas_own, normals_own, ff, vars_own, iterations: int,
                          exact: bool = False):
    """Rodinia euler on this rank's element slab with the fused peer-memory
    exchange: per RK stage one stage kernel (waits on the arrival counter)
    and one push kernel (stores the halo values into the peers' arrays, counts
    an arrival on each) -- no NCCL call and no host round trip.  Returns this
    rank's own columns (a copy).  Bit-identical to the single-device run."""
    import torch
    plan, lib = slabs.plan, slabs.lib
    n_own, n_loc = plan["n_own"], plan["n_loc"]
    stream = torch.cuda.current_stream().cuda_stream
    key = ("_nbrs", str(vars_own.device))
    if key not in plan:
        plan[key] = torch.as_tensor(plan["neighbors"]).to(vars_own.device)
    nbrs = plan[key]
    V = slabs.array(0)
    V[:, :n_own] = vars_own
    slabs.push(0, stream)  # V's halo values into the peers' V arrays
    pushes = 1
    for _ in range(iterations):
        for j, (cb, db) in enumerate(((0, 1), (1, 2), (2, 0))):
            target = slabs.epoch + pushes  # every source has pushed `pushes` times this call
            rc = lib.jb_euler_stage_p2p_f32(n_own, n_loc, j, areas_own.data_ptr(), nbrs.data_ptr(),
                                            normals_own.data_ptr(), ff.data_ptr(), slabs.buf(cb), slabs.buf(0),
                                            slabs.buf(db), slabs.flags(), slabs.srcmask, target, int(exact),
                                            stream)
            if rc:
                raise RuntimeError(f"euler_stage_p2p: {_lib.last_error()}")
            slabs.push(db, stream)
            pushes += 1
    slabs.epoch += pushes
    return V[:, :n_own].clone()


class CudaEulerBackend:
    """libjunob200's slab stage kernel on device tensors (NCCL exchanges).
    exact=True: the bit-exact stage (else the tolerance mode of jb_euler_f32;
    either way a sharded run is bit-identical to the single-device run of the
    same mode, since CFD has no reductions)."""

    def __init__(self, exact: bool = False):
        import torch
        self.torch = torch
        self.lib = _lib.load()
        self.exact = exact

    def to_device(self, a, like):
        return self.torch.as_tensor(a).to(like.device)

    def stage(self, n_own, n_loc, j, areas, nbrs, normals, ff, cur, old, dst):
        rc = self.lib.jb_euler_stage_f32(int(n_own), int(n_loc), int(j), areas.data_ptr(), nbrs.data_ptr(),
                                         normals.data_ptr(), ff.data_ptr(), cur.data_ptr(), old.data_ptr(),
                                         dst.data_ptr(), int(self.exact), self.torch.cuda.current_stream().cuda_stream)
        if rc:
            raise RuntimeError(f"euler_stage: {_lib.last_error()}")
