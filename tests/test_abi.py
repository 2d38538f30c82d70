"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/junob200.h declares, and the host layer validates arguments
the way the reference does before any device work."""
import ctypes

import numpy as np
import pytest

from paper_2503_10855_b200 import _lib


def test_header_declares_entries():
    syms = _lib.header_symbols()
    for want in ("jb_matmul_f32", "jb_edge_f32", "jb_cava_u8", "jb_srad_f32", "jb_euler_f32",
                 "jb_bfs", "jb_bp_train_f32", "jb_last_error", "jb_abi_version"):
        assert want in syms


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in _lib.header_symbols() if not hasattr(lib, s)]
    assert not missing, f"libjunob200.so lacks {missing}"


def test_abi_version_and_signatures():
    lib = _lib.load()
    assert lib.jb_abi_version() == 1
    for name in _lib.SIGNATURES:
        assert name in _lib.header_symbols()


def test_execute_validates_like_the_reference():
    import paper_2503_10855_b200 as jb
    a = np.zeros((4, 3), np.float32)
    b = np.zeros((3, 5), np.float32)
    with pytest.raises(jb.DynConstError):
        jb.execute("matmul", [4, -3, 5], [a, b])
    with pytest.raises(jb.DynConstError):
        jb.execute("matmul", [4, 3], [a, b])
    with pytest.raises(jb.RuntimeError_):
        jb.execute("matmul", [4, 4, 5], [a, b])
    with pytest.raises(jb.RuntimeError_):
        jb.execute("no_such_entry", [], [])


def test_oracle_execute_signature_parity():
    import inspect
    import paper_2503_10855_b200 as jb
    params = list(inspect.signature(jb.oracle_execute).parameters)
    assert params == ["module", "entry", "dyn_consts", "args", "max_steps"]


@pytest.mark.parametrize("frames,frame_px", [(1, 1), (2, 31), (3, 32), (2, 33), (4, 1000), (2, 8192 * 32 + 5),
                                             (1, 1080 * 1920)])
@pytest.mark.parametrize("threads", [1, 3, 0])
def test_bits_expand_host(frames, frame_px, threads):
    """jb_bits_expand_f32 (host code, no GPU): bit b of word w of a frame is
    pixel 32w+b -> 1.0f / 0.0f, ragged last words included, every output
    element written (sentinel-filled buffer)."""
    lib = _lib.load()
    fw = (frame_px + 31) // 32
    rng = np.random.default_rng(frame_px)
    words = rng.integers(0, 2 ** 32, size=(frames, fw), dtype=np.uint64).astype(np.uint32)
    bits = np.unpackbits(words.view(np.uint8).reshape(frames, fw * 4), axis=1, bitorder="little")
    want = bits[:, :frame_px].astype(np.float32)
    out = np.full((frames, frame_px), np.float32(7.0))
    assert lib.jb_bits_expand_f32(words.ctypes.data, frames, frame_px, out.ctypes.data, threads) == 0
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
    # an output that is not 16-byte aligned takes the unaligned stores
    buf = np.full(frames * frame_px + 1, np.float32(7.0))
    assert lib.jb_bits_expand_f32(words.ctypes.data, frames, frame_px, buf[1:].ctypes.data, threads) == 0
    assert np.array_equal(buf[1:].reshape(frames, frame_px), want)


@pytest.mark.filterwarnings("ignore:This process:DeprecationWarning")
def test_bits_expand_after_fork():
    """The host thread pool is per process: a forked child (multiprocessing
    'fork', torchrun helpers) gets its own workers instead of waiting on the
    parent's, which do not exist in the child."""
    import multiprocessing as mp
    lib = _lib.load()
    words = np.full((2, 64), 0xA5A5A5A5, np.uint32)
    out = np.zeros((2, 2048), np.float32)
    assert lib.jb_bits_expand_f32(words.ctypes.data, 2, 2048, out.ctypes.data, 0) == 0  # parent pool exists

    def child(q):
        o = np.zeros((2, 2048), np.float32)
        rc = _lib.load().jb_bits_expand_f32(words.ctypes.data, 2, 2048, o.ctypes.data, 0)
        q.put((rc, float(o.sum())))

    ctx = mp.get_context("fork")
    q = ctx.Queue()
    p = ctx.Process(target=child, args=(q,))
    p.start()
    p.join(60)
    assert not p.is_alive(), "the child's expansion hung"
    rc, total = q.get(timeout=5)
    assert rc == 0 and total == float(out.sum()) == 2 * 2048 / 2
