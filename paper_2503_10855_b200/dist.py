"""Multi-GPU partitioning of the Juno benchmarks.

One process per GPU (torch.distributed; NCCL over NVLink on the B200 box,
gloo in the CPU tests).  What shards and how:

  edge, CAVA   frames split across ranks, no collective      (shard_frames)
  matmul       row blocks of A and C, B replicated once       (row_block, matmul_row_blocks)
  SRAD         row slabs with 1 halo row above / 2 below; per iteration an
               allreduce of the f64 (sum, sum^2) pair and a halo exchange of
               the image rows                                 (srad_distributed)
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


def matmul_row_blocks(a_rows, b, group=None, src: int = 0):
    """C[rows] = A[rows] @ B on this rank; B is broadcast from `src` once."""
    import torch.distributed as dist

    from .api import matmul
    if dist.is_initialized():
        dist.broadcast(b, src=src, group=group)
    return matmul(a_rows, b)


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
    def step(self, J_ext, own_lo: int, own_hi: int, q0, lam: float, compress: bool): ...  # -> (out_own, sums)
    def q0(self, sums, npx: int): ...                              # -> q0 (backend tensor)
    def cat_rows(self, parts): ...


def _halo_exchange(J_own, rank: int, world: int, group, backend):
    """Return the extended slab [north 1 | own | south 2] (edges trimmed)."""
    import torch
    import torch.distributed as dist
    cols = J_own.shape[1]
    ops, north, south = [], None, None
    if rank > 0:
        north = torch.empty((1, cols), dtype=J_own.dtype, device=J_own.device)
        ops.append(dist.P2POp(dist.irecv, north, rank - 1, group))
        ops.append(dist.P2POp(dist.isend, J_own[:2].contiguous(), rank - 1, group))
    if rank < world - 1:
        south = torch.empty((2, cols), dtype=J_own.dtype, device=J_own.device)
        ops.append(dist.P2POp(dist.irecv, south, rank + 1, group))
        ops.append(dist.P2POp(dist.isend, J_own[-1:].contiguous(), rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    parts = [p for p in (north, J_own, south) if p is not None]
    return backend.cat_rows(parts)


def srad_distributed(image_own, niter: int, lam: float, rows: int, cols: int, backend: SradBackend,
                     group=None):
    """Row-slab SRAD across the ranks of `group`.  `image_own` holds this
    rank's rows (srad_slab(...)[r0:r1]); returns this rank's output rows."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    plan = srad_slab(rows, world, rank)
    assert image_own.shape[0] == plan["r1"] - plan["r0"] and image_own.shape[1] == cols
    npx = rows * cols
    if niter == 0:
        out, _ = backend.extract(image_own, compress=True)
        return out
    J, sums = backend.extract(image_own, compress=False)
    if world > 1:
        dist.all_reduce(sums, group=group)
    q0 = backend.q0(sums, npx)
    for it in range(niter):
        last = it + 1 == niter
        J_ext = _halo_exchange(J, rank, world, group, backend) if world > 1 else J
        J, sums = backend.step(J_ext, plan["own_lo"], plan["own_hi"], q0, lam, compress=last)
        if not last:
            if world > 1:
                dist.all_reduce(sums, group=group)
            q0 = backend.q0(sums, npx)
    return J


class CudaSradBackend:
    """libjunob200 slab kernels on device tensors (NCCL collectives)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.lib = _lib.load()

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

    def step(self, J_ext, own_lo, own_hi, q0, lam, compress):
        t = self.torch
        out = t.empty((own_hi - own_lo, J_ext.shape[1]), dtype=t.float32, device=J_ext.device)
        sums = t.zeros(2, dtype=t.float64, device=J_ext.device)
        self._chk(self.lib.jb_srad_slab_step_f32(J_ext.shape[0], J_ext.shape[1], own_lo, own_hi,
                                                 J_ext.data_ptr(), out.data_ptr(), q0.data_ptr(), float(lam),
                                                 sums.data_ptr(), int(compress), self._s()), "srad_slab_step")
        return out, sums

    def q0(self, sums, npx):
        q = self.torch.empty(1, dtype=self.torch.float32, device=sums.device)
        self._chk(self.lib.jb_srad_q0_f32(sums.data_ptr(), int(npx), q.data_ptr(), self._s()), "srad_q0")
        return q

    def cat_rows(self, parts):
        return self.torch.cat(parts, dim=0).contiguous()
