"""ctypes front-end of the CPU restatement (oracle/juno_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package.  Every function mirrors one Juno entry point and takes/returns
numpy arrays with the reference's boundary layout (C-contiguous row-major,
``skiff/types.py:147-159``).  The semantics contract is documented in
juno_oracle.c's header and DESIGN.md §parity.

Pinning: matmul and BFS are checked bit-for-bit against the reference
interpreter ``oracle_execute`` (runtime/oracle.py:28-32) through
tests/golden/*.npz (made by oracle/gen_golden.py); the gaussian, laplacian,
reject, max-gradient, SRAD-coefficient, CAVA scale/transform and BP
adjust-weights stages are pinned the same way with oracle-friendly Juno
fixtures.  oracle/gen_golden_fixed.py runs the same interpreter with its
Appendix A dependents defect fixed and pins the accumulator-form programs
and the stages around sqrt (CAVA demosaic, median, gamut, tone map; CFD step
factor and flux; SRAD q0 statistics; BP error stages): radicands and sums
are Juno programs, the IEEE sqrt between them numpy's.  What stays unpinned
is the transcendental itself (sqrt/exp/log: IEEE or f64-rounded on both
sides) and the f64 exp/log of SRAD's extract/compress and
BP's squash.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libjunooracle.so")
_lib = None

_f32p = ctypes.POINTER(ctypes.c_float)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _p(a: np.ndarray, ty):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ty)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def max_threads() -> int:
    return int(lib().jo_max_threads())


def set_threads(n: int) -> None:
    lib().jo_set_threads(int(n))


# -- matmul -------------------------------------------------
def matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a, b = _f32(a), _f32(b)
    n, m = a.shape
    m2, l = b.shape
    assert m == m2
    out = np.empty((n, l), np.float32)
    lib().jo_matmul_f32(_i64(n), _i64(m), _i64(l), _p(a, _f32p), _p(b, _f32p),
                        _p(out, _f32p))
    return out


# -- edge detection ------------------------------------------------------------
def edge_frame(img, gf, st, sx, sy, theta, stages: bool = False):
    img, gf, st, sx, sy = map(_f32, (img, gf, st, sx, sy))
    n, m = img.shape
    out = np.empty_like(img)
    if stages:
        sm, lp, zc, gr = (np.empty_like(img) for _ in range(4))
        mx = np.zeros(1, np.float32)
        ptrs = [_p(x, _f32p) for x in (sm, lp, zc, gr, mx)]
    else:
        ptrs = [None] * 5
    lib().jo_edge_frame_f32(_i64(n), _i64(m), _i64(gf.shape[0]), _i64(st.shape[0]),
                            _i64(sx.shape[0]), _p(img, _f32p), _p(gf, _f32p),
                            _p(st, _f32p), _p(sx, _f32p), _p(sy, _f32p),
                            ctypes.c_float(float(theta)), _p(out, _f32p), *ptrs)
    if stages:
        return dict(out=out, smoothed=sm, laplacian=lp, zero_crossings=zc,
                    gradient=gr, max_gradient=np.float32(mx[0]))
    return out


def edge(batch_imgs, gf, st, sx, sy, theta) -> np.ndarray:
    x = _f32(batch_imgs)
    b, n, m = x.shape
    gf, st, sx, sy = map(_f32, (gf, st, sx, sy))
    out = np.empty_like(x)
    lib().jo_edge_f32(_i64(b), _i64(n), _i64(m), _i64(gf.shape[0]), _i64(st.shape[0]),
                      _i64(sx.shape[0]), _p(x, _f32p), _p(gf, _f32p), _p(st, _f32p),
                      _p(sx, _f32p), _p(sy, _f32p), ctypes.c_float(float(theta)),
                      _p(out, _f32p))
    return out


# -- CAVA -------------------------------------------------------------------------
def cava_frame(raw, tstw, ctrl, wts, coefs, tmap, stages: bool = False):
    raw = np.ascontiguousarray(raw, dtype=np.uint8)
    tstw, ctrl, wts, coefs, tmap = map(_f32, (tstw, ctrl, wts, coefs, tmap))
    _, r, c = raw.shape
    out = np.empty_like(raw)
    if stages:
        dm, dn, gm = (np.empty(raw.shape, np.float32) for _ in range(3))
        ptrs = [_p(x, _f32p) for x in (dm, dn, gm)]
    else:
        ptrs = [None] * 3
    lib().jo_cava_frame_u8(_i64(r), _i64(c), _i64(ctrl.shape[0]), _p(raw, _u8p),
                           _p(tstw, _f32p), _p(ctrl, _f32p), _p(wts, _f32p),
                           _p(coefs, _f32p), _p(tmap, _f32p), _p(out, _u8p), *ptrs)
    if stages:
        return dict(out=out, demosaic=dm, denoise=dn, gamut=gm)
    return out


def cava(raw_batch, tstw, ctrl, wts, coefs, tmap) -> np.ndarray:
    raw = np.ascontiguousarray(raw_batch, dtype=np.uint8)
    tstw, ctrl, wts, coefs, tmap = map(_f32, (tstw, ctrl, wts, coefs, tmap))
    b, _, r, c = raw.shape
    out = np.empty_like(raw)
    lib().jo_cava_u8(_i64(b), _i64(r), _i64(c), _i64(ctrl.shape[0]), _p(raw, _u8p),
                     _p(tstw, _f32p), _p(ctrl, _f32p), _p(wts, _f32p), _p(coefs, _f32p),
                     _p(tmap, _f32p), _p(out, _u8p))
    return out


# -- SRAD -----------------------------------------------------------------------
def srad(image, niter: int, lam: float, return_q0: bool = False, acc64: bool = True):
    """acc64: q0^2 from f64 sums rounded once (the GPU contract); False:
    Rodinia's sequential f32 sums."""
    img = _f32(image)
    rows, cols = img.shape
    out = np.empty_like(img)
    q0 = np.zeros(max(int(niter), 1), np.float32)
    lib().jo_srad_f32_acc(_i64(rows), _i64(cols), _i64(niter), ctypes.c_float(lam),
                          _p(img, _f32p), _p(out, _f32p), _p(q0, _f32p), ctypes.c_int(1 if acc64 else 0))
    return (out, q0[:niter]) if return_q0 else out


# -- CFD / Euler -------------------------------------------------------------------
def euler(areas, nbrs, normals, ff, variables, iterations: int) -> np.ndarray:
    areas, normals, ff = _f32(areas), _f32(normals), _f32(ff)
    nbrs = np.ascontiguousarray(nbrs, dtype=np.int32)
    v = _f32(variables).copy()
    nelr = areas.shape[0]
    lib().jo_euler_f32(_i64(nelr), _i64(iterations), _p(areas, _f32p), _p(nbrs, _i32p),
                       _p(normals, _f32p), _p(ff, _f32p), _p(v, _f32p))
    return v


def euler_step_factor(variables, areas) -> np.ndarray:
    variables, areas = _f32(variables), _f32(areas)
    nelr = areas.shape[0]
    sf = np.empty(nelr, np.float32)
    lib().jo_euler_step_factor(_i64(nelr), _p(variables, _f32p), _p(areas, _f32p),
                               _p(sf, _f32p))
    return sf


def euler_flux(nbrs, normals, ff, variables) -> np.ndarray:
    normals, ff, variables = _f32(normals), _f32(ff), _f32(variables)
    nbrs = np.ascontiguousarray(nbrs, dtype=np.int32)
    nelr = nbrs.shape[1]
    fl = np.empty((5, nelr), np.float32)
    lib().jo_euler_flux(_i64(nelr), _p(nbrs, _i32p), _p(normals, _f32p), _p(ff, _f32p),
                        _p(variables, _f32p), _p(fl, _f32p))
    return fl


# -- BFS --------------------------------------------------------------------------
def bfs(starting, nedges, edges, source: int) -> np.ndarray:
    s = np.ascontiguousarray(starting, dtype=np.uint32)
    ne = np.ascontiguousarray(nedges, dtype=np.uint32)
    e = np.ascontiguousarray(edges, dtype=np.uint32)
    n = s.shape[0]
    cost = np.empty(n, np.int32)
    lib().jo_bfs(_i64(n), _i64(e.shape[0]), _p(s, _u32p), _p(ne, _u32p),
                 _p(e if e.size else np.zeros(1, np.uint32), _u32p),
                 ctypes.c_uint32(source), _p(cost, _i32p))
    return cost


# -- backprop -------------------------------------------------------------------------
def bp_train(input_units, in_w, hid_w, target, in_prev_w, hid_prev_w, acc64=True):
    """One bpnn_train step.  Returns a dict; arrays are fresh copies."""
    x = _f32(input_units).copy()
    iw, hw = _f32(in_w).copy(), _f32(hid_w).copy()
    ipw, hpw = _f32(in_prev_w).copy(), _f32(hid_prev_w).copy()
    t = _f32(target)
    n_in, n_hid = iw.shape[0] - 1, iw.shape[1] - 1
    n_out = hw.shape[1] - 1
    hidden = np.zeros(n_hid + 1, np.float32)
    output = np.zeros(n_out + 1, np.float32)
    d_o = np.zeros(n_out + 1, np.float32)
    d_h = np.zeros(n_hid + 1, np.float32)
    errs = np.zeros(2, np.float32)
    lib().jo_bp_train(_i64(n_in), _i64(n_hid), _i64(n_out), _p(x, _f32p), _p(iw, _f32p),
                      _p(hw, _f32p), _p(t, _f32p), _p(ipw, _f32p), _p(hpw, _f32p),
                      _p(hidden, _f32p), _p(output, _f32p), _p(d_o, _f32p), _p(d_h, _f32p),
                      _p(errs, _f32p), ctypes.c_int(1 if acc64 else 0))
    return dict(input=x, input_weights=iw, hidden_weights=hw, input_prev_weights=ipw,
                hidden_prev_weights=hpw, hidden=hidden, output=output, delta_o=d_o,
                delta_h=d_h, out_err=np.float32(errs[0]), hid_err=np.float32(errs[1]))


# -- stage functions (golden-vector pinning) -------------------------------------
def srad_iter(J, q0sqr: float, lam: float) -> np.ndarray:
    """One SRAD iteration (coefficient + update) for a given q0^2."""
    J = _f32(J).copy()
    rows, cols = J.shape
    tmp = [np.empty_like(J) for _ in range(5)]
    lib().jo_srad_iter(_i64(rows), _i64(cols), ctypes.c_float(q0sqr), ctypes.c_float(lam),
                       _p(J, _f32p), *[_p(t, _f32p) for t in tmp])
    return J


def srad_q0sqr(J) -> np.float32:
    J = _f32(J)
    fn = lib().jo_srad_q0sqr
    fn.restype = ctypes.c_float
    return np.float32(fn(_i64(J.size), _p(J, _f32p)))


def bp_layer_sums(l1, conn, acc64=False) -> np.ndarray:
    l1, conn = _f32(l1), _f32(conn)
    n1, n2 = conn.shape[0] - 1, conn.shape[1] - 1
    out = np.empty(n2 + 1, np.float32)
    lib().jo_bp_layer_sums(_i64(n1), _i64(n2), _p(l1, _f32p), _p(conn, _f32p), _p(out, _f32p),
                           ctypes.c_int(1 if acc64 else 0))
    return out


def bp_adjust_weights(delta, ly, w, oldw):
    """Returns (w', oldw'); ly[0] is forced to the bias 1.0 like Rodinia."""
    delta, ly = _f32(delta), _f32(ly).copy()
    w, oldw = _f32(w).copy(), _f32(oldw).copy()
    nly, nd = w.shape[0] - 1, w.shape[1] - 1
    lib().jo_bp_adjust_weights(_p(delta, _f32p), _i64(nd), _p(ly, _f32p), _i64(nly), _p(w, _f32p),
                               _p(oldw, _f32p))
    return w, oldw


def cava_stage(name: str, *arrays, P: int = 0):
    """Run one CAVA stage on [3,R,C] planes: scale | demosaic | denoise |
    transform | gamut | tonemap_descale."""
    L = lib()
    if name == "scale":
        raw = np.ascontiguousarray(arrays[0], np.uint8)
        _, R, C = raw.shape
        out = np.empty(raw.shape, np.float32)
        L.jo_cava_scale(_i64(R), _i64(C), _p(raw, _u8p), _p(out, _f32p))
        return out
    x = _f32(arrays[0])
    _, R, C = x.shape
    N = R * C
    if name in ("demosaic", "denoise"):
        out = np.empty_like(x)
        getattr(L, f"jo_cava_{name}")(_i64(R), _i64(C), _p(x, _f32p), _p(out, _f32p))
        return out
    if name == "transform":
        t = _f32(arrays[1])
        out = np.empty_like(x)
        L.jo_cava_transform(_i64(N), _p(x, _f32p), _p(t, _f32p), _p(out, _f32p))
        return out
    if name == "gamut":
        ctrl, wts, coefs = map(_f32, arrays[1:4])
        out = np.empty_like(x)
        L.jo_cava_gamut(_i64(N), _i64(ctrl.shape[0]), _p(x, _f32p), _p(ctrl, _f32p), _p(wts, _f32p),
                        _p(coefs, _f32p), _p(out, _f32p))
        return out
    if name == "tonemap_descale":
        tm = _f32(arrays[1])
        out = np.empty(x.shape, np.uint8)
        L.jo_cava_tonemap_descale(_i64(N), _p(x, _f32p), _p(tm, _f32p), _p(out, _u8p))
        return out
    raise ValueError(name)


# -- SRAD slab helpers (tests of paper_2503_10855_b200.dist) -------------------
def srad_extract(image, compress=False) -> np.ndarray:
    img = _f32(image)
    out = np.empty_like(img)
    lib().jo_srad_extract(_i64(img.size), _p(img, _f32p), _p(out, _f32p), ctypes.c_int(int(compress)))
    return out


def srad_sums(J) -> np.ndarray:
    J = _f32(J)
    out = np.zeros(2, np.float64)
    lib().jo_srad_sums(_i64(J.size), _p(J, _f32p), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def srad_compress(J) -> np.ndarray:
    J = _f32(J)
    out = np.empty_like(J)
    lib().jo_srad_compress(_i64(J.size), _p(J, _f32p), _p(out, _f32p))
    return out
