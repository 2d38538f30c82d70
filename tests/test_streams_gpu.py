"""Concurrent calls on different streams of one device.

The library's per-call state -- the edge filters in the device's
``__constant__`` bank, the scratch arena, matmul's tensor-map and graph
caches -- must not let two streams' calls corrupt each other: the scratch is
per (device, stream), and a call on another stream than the previous edge
call first waits for that call's kernels before it rewrites the filter bank.
Each stream's results are checked against the oracle after interleaved,
unsynchronised launches.
"""
import numpy as np
import pytest

from paper_2503_10855_b200 import _lib
from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def test_edge_two_streams_different_filters(jb, oracle):
    import torch
    lib = _lib.load()
    g1, st, sx, sy, th = W.edge_filters()
    rng = np.random.default_rng(2)
    g2 = rng.uniform(0.01, 0.05, (7, 7)).astype(np.float32)  # another filter: not mirror-symmetric
    xa = np.stack([W.edge_frame(270, 480, seed=s) for s in range(6)])
    xb = np.stack([W.edge_frame(270, 480, seed=50 + s) for s in range(6)])
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    fa = [dev(a) for a in (g1, st, sx, sy)]
    fb = [dev(a) for a in (g2, st, sx, sy)]
    da, db = dev(xa), dev(xb)
    torch.cuda.synchronize()
    outs_a, outs_b = [], []
    for _ in range(4):
        for stream, x, flt, outs in ((sa, da, fa, outs_a), (sb, db, fb, outs_b)):
            o = torch.empty_like(x)
            with torch.cuda.stream(stream):
                rc = lib.jb_edge_f32(6, 270, 480, 7, 3, 3, x.data_ptr(), *[t.data_ptr() for t in flt], float(th),
                                     o.data_ptr(), stream.cuda_stream)
            assert rc == 0, _lib.last_error()
            outs.append(o)
    torch.cuda.synchronize()
    ra = oracle.edge(xa, g1, st, sx, sy, th)
    rb = oracle.edge(xb, g2, st, sx, sy, th)
    for o in outs_a:
        assert np.array_equal(_bits(o.cpu().numpy()), _bits(ra))
    for o in outs_b:
        assert np.array_equal(_bits(o.cpu().numpy()), _bits(rb))


def test_srad_and_matmul_two_streams(jb, oracle):
    """Per-stream scratch: SRAD's statistics/ping-pong scratch and matmul's
    operands on two streams at once."""
    import torch
    lib = _lib.load()
    img1, img2 = W.srad_image(512, 384, seed=1), W.srad_image(512, 384, seed=2)
    a1, b1 = W.matmul_inputs(512, 256, 384, seed=3)
    a2, b2 = W.matmul_inputs(512, 256, 384, seed=4)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    d = {k: dev(v) for k, v in dict(img1=img1, img2=img2, a1=a1, b1=b1, a2=a2, b2=b2).items()}
    torch.cuda.synchronize()
    res = []
    for it in range(3):
        for s, img, a, b in ((s1, "img1", "a1", "b1"), (s2, "img2", "a2", "b2")):
            out = torch.empty_like(d[img])
            q0 = torch.empty(5, dtype=torch.float32, device="cuda")
            c = torch.empty((512, 384), dtype=torch.float32, device="cuda")
            with torch.cuda.stream(s):
                assert lib.jb_srad_f32(512, 384, 5, 0.5, d[img].data_ptr(), out.data_ptr(), q0.data_ptr(),
                                       s.cuda_stream) == 0, _lib.last_error()
                assert lib.jb_matmul_f32(512, 256, 384, d[a].data_ptr(), d[b].data_ptr(), c.data_ptr(),
                                         s.cuda_stream) == 0, _lib.last_error()
            res.append((img, a, b, out, c))
    torch.cuda.synchronize()
    want = {"img1": jb.srad(5, 0.5, img1), "img2": jb.srad(5, 0.5, img2)}
    mm = {"a1": jb.matmul(a1, b1), "a2": jb.matmul(a2, b2)}
    for img, a, b, out, c in res:
        assert np.array_equal(_bits(out.cpu().numpy()), _bits(want[img]))
        assert np.array_equal(_bits(c.cpu().numpy()), _bits(mm[a]))
