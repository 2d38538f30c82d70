"""Multi-rank host logic (paper_2503_10855_b200.dist) on CPU with gloo,
world_size 2 and 3: the same slab/halo/allreduce driver the GPU path runs,
with the oracle restatement as the per-slab compute (test-only backend)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_10855_b200 import dist as D


def test_partition_covers_exactly():
    for n in (1, 7, 256, 1000):
        for w in (1, 2, 3, 8):
            spans = [D.partition(n, w, r) for r in range(w)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == n
            for (a, ca), (b, _) in zip(spans, spans[1:]):
                assert a + ca == b
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def test_srad_slab_plan_halos():
    p = D.srad_slab(100, 4, 0)
    assert (p["r0"], p["e0"], p["own_lo"]) == (0, 0, 0) and p["e1"] == p["r1"] + 2
    p = D.srad_slab(100, 4, 3)
    assert p["e1"] == 100 and p["e0"] == p["r0"] - 1 and p["own_lo"] == 1
    with pytest.raises(ValueError):
        D.srad_slab(5, 4, 0)


class OracleSradBackend:
    """CPU stand-in for CudaSradBackend built on the C restatement."""

    def __init__(self):
        from oracle import oracle
        self.o = oracle

    def extract(self, image_own, compress):
        a = image_own.numpy()
        J = self.o.srad_extract(a, compress=compress)
        return torch.from_numpy(J), torch.from_numpy(self.o.srad_sums(J))

    def empty_rows(self, n, cols, like):
        return torch.empty((n, cols), dtype=torch.float32)

    def step(self, J_ext, own_lo, own_hi, q0, lam, compress, out=None):
        J = self.o.srad_iter(J_ext.numpy(), float(q0.item()), float(lam))[own_lo:own_hi]
        if compress:
            res, sums = torch.from_numpy(self.o.srad_compress(J)), torch.zeros(2, dtype=torch.float64)
        else:
            res, sums = torch.from_numpy(np.ascontiguousarray(J)), torch.from_numpy(self.o.srad_sums(J))
        if out is not None:
            out.copy_(res)
            res = out
        return res, sums

    def q0(self, sums, npx):
        s, s2 = float(sums[0]), float(sums[1])
        mean = s / npx
        var = s2 / npx - mean * mean
        return torch.tensor([np.float32(var / (mean * mean))])

    def cat_rows(self, parts):
        return torch.cat(parts, dim=0).contiguous()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def _run(world, fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


ROWS, COLS, NITER = 41, 23, 4


def _srad_rank(rank, world):
    from paper_2503_10855_b200 import workloads as W
    img = W.srad_image(ROWS, COLS, seed=5)
    plan = D.srad_slab(ROWS, world, rank)
    own = torch.from_numpy(np.ascontiguousarray(img[plan["r0"]:plan["r1"]]))
    return D.srad_distributed(own, NITER, 0.5, ROWS, COLS, OracleSradBackend()).numpy()


def _frames_rank(rank, world):
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    g, st, sx, sy, th = W.edge_filters()
    batch = W.edge_batch(5, 30, 44, seed=3, distinct=5)
    f0, cnt = D.shard_frames(5, world, rank)
    out = torch.from_numpy(oracle.edge(batch[f0:f0 + cnt], g, st, sx, sy, th))
    sizes = [D.shard_frames(5, world, r)[1] for r in range(world)]
    # uneven shards: gather through a padded buffer
    pad = torch.zeros((max(sizes), 30, 44))
    pad[:cnt] = out
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)]).numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_srad_row_slabs_match_single_device(world):
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    parts = _run(world, _srad_rank)
    got = np.concatenate(parts)
    ref = oracle.srad(W.srad_image(ROWS, COLS, seed=5), NITER, 0.5)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_frame_sharding_gathers_the_batch():
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    g, st, sx, sy, th = W.edge_filters()
    ref = oracle.edge(W.edge_batch(5, 30, 44, seed=3, distinct=5), g, st, sx, sy, th)
    outs = _run(2, _frames_rank)
    for o in outs:
        assert np.array_equal(o.view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------------------ CFD
class OracleEulerBackend:
    """CPU stand-in for CudaEulerBackend: the slab stage from the C
    restatement's flux / step-factor on the slab-local arrays (halo columns
    padded as walls; only the own columns are kept)."""

    def __init__(self):
        from oracle import oracle
        self.o = oracle

    def to_device(self, a, like):
        return torch.as_tensor(a)

    def stage(self, n_own, n_loc, j, areas, nbrs, normals, ff, cur, old, dst):
        nb = np.full((4, n_loc), -1, np.int32)
        nb[:, :n_own] = nbrs.numpy()
        nr = np.zeros((4, 3, n_loc), np.float32)
        nr[:, :, :n_own] = normals.numpy()
        fl = self.o.euler_flux(nb, nr, ff.numpy(), np.ascontiguousarray(cur.numpy()))[:, :n_own]
        o = np.ascontiguousarray(old.numpy()[:, :n_own])
        sf = self.o.euler_step_factor(o, areas.numpy())
        factor = sf / np.float32(4 - j)  # RK + 1 - j
        dst[:, :n_own] = torch.from_numpy((o + factor[None, :] * fl).astype(np.float32))


MESH_W, MESH_H, CFD_ITERS = 12, 9, 2


def _euler_rank(rank, world):
    from paper_2503_10855_b200 import workloads as W
    areas, nb, normals, ff, v = W.euler_mesh(MESH_W, MESH_H, seed=3)
    plan = D.euler_plan(nb, world, rank)
    e0, e1 = plan["e0"], plan["e1"]
    vl = torch.zeros((5, plan["n_loc"]), dtype=torch.float32)
    vl[:, :plan["n_own"]] = torch.from_numpy(v[:, e0:e1])
    out = D.euler_distributed(plan, torch.from_numpy(np.ascontiguousarray(areas[e0:e1])),
                              torch.from_numpy(np.ascontiguousarray(normals[:, :, e0:e1])),
                              torch.from_numpy(ff), vl, CFD_ITERS, OracleEulerBackend())
    return out.numpy().copy()


def test_euler_plan_structured_mesh_halo_is_one_row():
    from paper_2503_10855_b200 import workloads as W
    _, nb, _, _, _ = W.euler_mesh(MESH_W, MESH_H)
    p = D.euler_plan(nb, 3, 1)
    assert p["n_loc"] - p["n_own"] == 2 * MESH_W  # one mesh row above and below
    assert sorted(p["recv"]) == [0, 2] and sorted(p["send"]) == [0, 2]
    assert all(len(ix) == MESH_W for ix in p["send"].values())
    loc = p["neighbors"]
    assert loc.min() >= -2 and loc.max() < p["n_loc"]


@pytest.mark.parametrize("world", [2, 3])
def test_euler_element_slabs_match_single_device(world):
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    areas, nb, normals, ff, v = W.euler_mesh(MESH_W, MESH_H, seed=3)
    ref = oracle.euler(areas, nb, normals, ff, v, CFD_ITERS)
    got = np.concatenate(_run(world, _euler_rank), axis=1)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


# --------------------------------------------------------- matmul / CAVA
MM_N, MM_M, MM_L = 37, 16, 24


def _matmul_rank(rank, world):
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    a, b = W.matmul_inputs(MM_N, MM_M, MM_L, seed=4)
    # only the source rank starts with B: the others receive it once
    bt = torch.from_numpy(b) if rank == 0 else torch.zeros((MM_M, MM_L), dtype=torch.float32)
    mb = D.MatmulRowBlocks(bt, MM_N, mm=lambda x, y: torch.from_numpy(oracle.matmul(x.numpy(), y.numpy())))
    a_own = torch.from_numpy(np.ascontiguousarray(mb.own_rows(a)))
    c1 = mb(a_own)
    c2 = mb(a_own)           # a second call: no further broadcast
    assert torch.equal(c1, c2) and mb.broadcasts == 1
    return c1.numpy(), mb.gather(c1).numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_matmul_row_blocks_match_single_device(world):
    """Row blocks of A and C with B broadcast once: the concatenated blocks
    (and the all-gathered C on every rank) are bit-identical to the
    single-device oracle (rows of the sequential-k product do not interact)."""
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    a, b = W.matmul_inputs(MM_N, MM_M, MM_L, seed=4)
    ref = oracle.matmul(a, b)
    outs = _run(world, _matmul_rank)
    got = np.concatenate([o[0] for o in outs])
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    for _, full in outs:
        assert np.array_equal(full.view(np.uint32), ref.view(np.uint32))


def _cava_rank(rank, world):
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    raw = W.cava_raw(5, 20, 34, seed=2)
    params = W.cava_params(16)
    f0, cnt = D.shard_frames(5, world, rank)
    out = torch.from_numpy(oracle.cava(raw[f0:f0 + cnt], *params))
    sizes = [D.shard_frames(5, world, r)[1] for r in range(world)]
    pad = torch.zeros((max(sizes), 3, 20, 34), dtype=torch.uint8)
    pad[:cnt] = out
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)]).numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_cava_frame_sharding_gathers_the_batch(world):
    from oracle import oracle
    from paper_2503_10855_b200 import workloads as W
    raw = W.cava_raw(5, 20, 34, seed=2)
    ref = oracle.cava(raw, *W.cava_params(16))
    for o in _run(world, _cava_rank):
        assert np.array_equal(o, ref)
