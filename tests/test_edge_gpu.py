"""edge_detection on the B200 vs the oracle restatement: bit-exact."""
import numpy as np
import pytest

from conftest import golden
from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    assert a.shape == b.shape
    diff = np.count_nonzero(a.view(np.uint32) != b.view(np.uint32))
    assert diff == 0, f"{diff} of {a.size} values differ"


@pytest.mark.parametrize("name", ["edge_12x16_g7", "edge_9x11_g3"])
def test_edge_matches_golden(jb, name):
    g = golden(name)
    out = jb.edge_detection(g["input"], g["gaussian"], g["structure"], g["sx"], g["sy"], g["theta"])
    _bits_equal(out, g["out"])
    st = jb.edge_detection_stages(g["input"], g["gaussian"], g["structure"], g["sx"], g["sy"], g["theta"])
    for k in ("smoothed", "laplacian", "zero_crossings", "gradient", "out"):
        _bits_equal(st[k], g[k])


def test_edge_gaussian_matches_fixed_interpreter_accumulator_form(jb):
    """The smoothed stage against skiff's interpreter (Appendix A defect
    fixed, oracle/gen_golden_fixed.py) running the gaussian in its natural
    scalar-accumulator form."""
    g = golden("fixed_interp")
    e = golden("edge_12x16_g7")
    st = jb.edge_detection_stages(g["edge_input"], g["gaussian"], e["structure"], e["sx"], e["sy"], e["theta"])
    _bits_equal(st["smoothed"], g["gaussian_acc"])


@pytest.mark.parametrize("shape", [(1, 60, 60), (2, 61, 59), (3, 128, 200), (1, 7, 5), (1, 1, 1),
                                   (2, 1080, 1920), (4, 121, 245),
                                   # more frames than packed-ring slots (slot reuse), and an odd
                                   # width (no TMA, scalar reject units)
                                   (12, 1080, 1920), (7, 1080, 1918),
                                   # 4K frames: the packed ring holds only 2 slots (reject lag 1)
                                   (3, 2160, 3840)])
def test_edge_fused_vs_oracle(jb, oracle, shape):
    b, n, m = shape
    g, st, sx, sy, th = W.edge_filters()
    x = np.stack([W.edge_frame(n, m, seed=s) for s in range(b)])
    out = jb.edge_detection(x, g, st, sx, sy, th)
    ref = oracle.edge(x, g, st, sx, sy, th)
    _bits_equal(out, ref)


@pytest.mark.parametrize("kind", ["random", "vsym_only", "perturbed_one_tap"])
def test_edge_gaussian_variants(jb, oracle, kind):
    """The packed gaussian shares mirrored products only when the filter is
    bitwise symmetric top to bottom; other 7x7 filters take the plain packed
    path.  Both must be bit-exact."""
    g, st, sx, sy, th = W.edge_filters()
    rng = np.random.default_rng(11)
    if kind == "random":
        g = (rng.random((7, 7), dtype=np.float32) / np.float32(49.0)).astype(np.float32)
    elif kind == "vsym_only":
        top = rng.random((4, 7), dtype=np.float32) / np.float32(49.0)
        g = np.concatenate([top, top[2::-1]]).astype(np.float32)   # rows i and 6-i equal
    else:
        g = g.copy()
        g[6, 3] = np.nextafter(g[6, 3], np.float32(1))              # breaks the symmetry by 1 ulp
    x = np.stack([W.edge_frame(200, 300, seed=s) for s in range(2)])
    _bits_equal(jb.edge_detection(x, g, st, sx, sy, th), oracle.edge(x, g, st, sx, sy, th))


def test_edge_exact_fallback_paths(jb, oracle):
    """Tiles whose data or filters violate the fast-path guard run the exact
    scalar path: negative pixels, subnormals, a non-unit structure and a
    non-power-of-two sobel must all stay bit-exact."""
    g, st, sx, sy, th = W.edge_filters()
    rng = np.random.default_rng(3)
    x = np.stack([W.edge_frame(130, 190, seed=9)] * 3)
    x[0, 10:20, 10:20] = -rng.random((10, 10), dtype=np.float32)   # negative pixels
    x[1, 70:75, 100:110] = np.float32(1e-39)                         # subnormals
    x[2, 0, 0] = np.float32(np.inf)                                  # non-finite
    x[2, 60:63, 90:93] = np.float32(-0.0)                            # negative zeros
    _bits_equal(jb.edge_detection(x, g, st, sx, sy, th), oracle.edge(x, g, st, sx, sy, th))
    st2 = st.copy(); st2[1, 1] = 0.5
    _bits_equal(jb.edge_detection(x[:2], g, st2, sx, sy, th), oracle.edge(x[:2], g, st2, sx, sy, th))
    sx2 = sx * np.float32(0.3)
    _bits_equal(jb.edge_detection(x[:2], g, st, sx2, sy, th), oracle.edge(x[:2], g, st, sx2, sy, th))
    # power-of-two but non-standard sobel: generic FFMA fast path
    sx4, sy4 = (-2 * sx).astype(np.float32), sy.T.copy()
    _bits_equal(jb.edge_detection(x[:2], g, st, sx4, sy4, th), oracle.edge(x[:2], g, st, sx4, sy4, th))


def test_edge_generic_sizes(jb, oracle):
    g5, st, sx, sy, th = W.edge_filters(gs=5)
    x = np.stack([W.edge_frame(50, 77, seed=4)])
    _bits_equal(jb.edge_detection(x, g5, st, sx, sy, th), oracle.edge(x, g5, st, sx, sy, th))
    st5 = np.ones((5, 5), np.float32)
    _bits_equal(jb.edge_detection(x, g5, st5, sx, sy, th), oracle.edge(x, g5, st5, sx, sy, th))


def test_edge_device_tensors_and_execute(jb, oracle):
    import torch
    g, st, sx, sy, th = W.edge_filters()
    x = W.edge_frame(96, 128, seed=5)
    dev = [torch.from_numpy(a).cuda() for a in (x, g, st, sx, sy)]
    out = jb.edge_detection(*dev, th)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    _bits_equal(out.cpu().numpy(), oracle.edge(x[None], g, st, sx, sy, th)[0])
    out2 = jb.execute("edge_detection", [96, 128, 7, 3, 3], [x, g, st, sx, sy, th])
    _bits_equal(out2, out.cpu().numpy())


@pytest.mark.parametrize("theta", [0.0, -0.0, -0.5, 1.0, 0.999, 3.0e38, float("inf"), float("nan")])
def test_edge_threshold_cases(jb, oracle, theta):
    """The in-kernel reject compares packed gradient bits against a per-frame
    threshold derived from theta * sqrt(max); it must agree with the oracle's
    float compare for every theta, including signed zero, inf and NaN."""
    g, st, sx, sy, _ = W.edge_filters()
    x = np.stack([W.edge_frame(130, 190, seed=s) for s in range(3)])
    th = np.float32(theta)
    _bits_equal(jb.edge_detection(x, g, st, sx, sy, th), oracle.edge(x, g, st, sx, sy, th))


def test_edge_pipelined_matches_single_call(jb):
    """The host-buffer pipelined entry returns exactly the single-call result
    (ragged last chunk included)."""
    import torch
    from paper_2503_10855_b200 import api
    g, st, sx, sy, th = W.edge_filters()
    x = np.stack([W.edge_frame(121, 245, seed=s) for s in range(7)])
    ref = jb.edge_detection(x, g, st, sx, sy, th)
    got = api.edge_detection_pipelined(torch.from_numpy(x).pin_memory(), g, st, sx, sy, th, chunk=3)
    _bits_equal(got.numpy(), ref)


def _pack_words(maps):
    """f32 maps [b, n, m] (0/1) -> u32 words [b, ceil(n*m/32)], bit b of word w = pixel 32w+b."""
    b = maps.shape[0]
    flat = (maps.reshape(b, -1) != 0).astype(np.uint8)
    fw = (flat.shape[1] + 31) // 32
    pad = np.zeros((b, fw * 32), np.uint8)
    pad[:, :flat.shape[1]] = flat
    return np.packbits(pad, axis=1, bitorder="little").view(np.uint32)


@pytest.mark.parametrize("shape,gs", [((3, 1080, 1920), 7), ((2, 61, 59), 7), ((5, 121, 245), 7), ((2, 7, 5), 7),
                                      ((3, 1080, 1918), 7), ((1, 1, 1), 7), ((2, 50, 77), 5)])
def test_edge_bits_entry_matches_f32_entry(jb, shape, gs):
    """jb_edge_bits_f32 writes exactly the bits of jb_edge_f32's maps: fused
    path (TMA and scalar reject units, ragged last word) and the generic
    per-stage path + packing kernel (gs=5)."""
    import torch
    from paper_2503_10855_b200 import _lib
    b, n, m = shape
    g, st, sx, sy, th = W.edge_filters(gs=gs)
    x = np.stack([W.edge_frame(n, m, seed=30 + s) for s in range(b)])
    d = [torch.from_numpy(a).cuda() for a in (x, g, st, sx, sy)]
    out = torch.empty_like(d[0])
    fw = (n * m + 31) // 32
    bits = torch.full((b, fw), -1, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    ptrs = [t.data_ptr() for t in d]
    assert lib.jb_edge_f32(b, n, m, gs, 3, 3, *ptrs, th, out.data_ptr(), s) == 0
    assert lib.jb_edge_bits_f32(b, n, m, gs, 3, 3, *ptrs, th, bits.data_ptr(), s) == 0, _lib.last_error()
    torch.cuda.synchronize()
    want = _pack_words(out.cpu().numpy())
    got = bits.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want), f"{np.count_nonzero(got != want)} words differ"
    assert np.count_nonzero(out.cpu().numpy()) > 0 or n * m < 64


def test_edge_pipelined_bits_equals_f32_transfer(jb):
    """The bit-packed D2H + host expansion returns the same f32 maps as the
    f32 transfer (several chunks, ragged last chunk, odd frame size)."""
    import torch
    from paper_2503_10855_b200 import api
    g, st, sx, sy, th = W.edge_filters()
    x = torch.from_numpy(np.stack([W.edge_frame(135, 241, seed=s) for s in range(9)])).pin_memory()
    a = api.edge_detection_pipelined(x, g, st, sx, sy, th, chunk=4, bits=False)
    b = api.edge_detection_pipelined(x, g, st, sx, sy, th, chunk=4, bits=True)
    _bits_equal(a.numpy(), b.numpy())
    assert a.numpy().any()
