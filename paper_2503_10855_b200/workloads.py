"""Seeded synthetic inputs of the shapes BASELINE.json names.

There is no network for datasets, so every benchmark runs on synthetic data
generated here with numpy; tests and bench.py share these generators so that
the oracle and the kernels see identical bytes.
"""

from __future__ import annotations

import numpy as np


# ------------------------------------------------------------------- matmul
def matmul_inputs(n=1024, m=1024, l=1024, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, (n, m)).astype(np.float32)
    b = rng.uniform(-1.0, 1.0, (m, l)).astype(np.float32)
    return a, b


# --------------------------------------------------------------------- edge
def edge_filters(gs=7, sigma=1.4, theta=0.1):
    """gaussian gs x gs (sigma, normalised), 3x3 structure of ones, sobel."""
    r = gs // 2
    ax = np.arange(-r, r + 1, dtype=np.float64)
    g = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2.0 * sigma * sigma))
    g = (g / g.sum()).astype(np.float32)
    structure = np.ones((3, 3), np.float32)
    sx = np.array([[-1, 0, 1], [-2, 0, 2], [-1, 0, 1]], np.float32)
    sy = np.array([[-1, -2, -1], [0, 0, 0], [1, 2, 1]], np.float32)
    return g, structure, sx, sy, np.float32(theta)


def edge_frame(n=1080, m=1920, seed=0, blobs=32, noise=0.02):
    """Sum of random gaussian blobs + gaussian noise, clipped to [0,1].
    Blobs are separable, so the frame is a (n x blobs) @ (blobs x m) product."""
    rng = np.random.default_rng(seed)
    cy = rng.uniform(0, n, blobs)
    cx = rng.uniform(0, m, blobs)
    sig = rng.uniform(0.02, 0.12, blobs) * min(n, m)
    amp = rng.uniform(0.2, 0.8, blobs)
    ys = np.arange(n)[:, None]
    xs = np.arange(m)[:, None]
    gy = np.exp(-((ys - cy[None, :]) ** 2) / (2 * sig[None, :] ** 2)) * amp[None, :]
    gx = np.exp(-((xs - cx[None, :]) ** 2) / (2 * sig[None, :] ** 2))
    img = gy @ gx.T
    img += noise * rng.standard_normal((n, m))
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def edge_batch(batch=256, n=1080, m=1920, seed=0, distinct=8):
    """`distinct` independently generated frames, each reused with a different
    cyclic shift so every frame of the batch has different content."""
    base = [edge_frame(n, m, seed + k) for k in range(min(distinct, batch))]
    out = np.empty((batch, n, m), np.float32)
    for f in range(batch):
        b = base[f % len(base)]
        shift = (f // len(base)) * 37
        out[f] = np.roll(b, shift=(shift % n, (3 * shift) % m), axis=(0, 1))
    return out


# --------------------------------------------------------------------- CAVA
def cava_params(P=16, seed=0):
    rng = np.random.default_rng(seed + 1)
    tstw = (np.eye(3) + 0.05 * rng.standard_normal((3, 3))).astype(np.float32)
    ctrl = rng.uniform(0.0, 1.0, (P, 3)).astype(np.float32)
    wts = (0.02 * rng.standard_normal((P, 3))).astype(np.float32)
    coefs = np.zeros((4, 3), np.float32)
    coefs[0] = 0.02 * rng.standard_normal(3)
    coefs[1:] = np.eye(3) + 0.02 * rng.standard_normal((3, 3))
    x = np.linspace(0.0, 1.0, 256)
    tmap = np.stack([x ** (1 / 2.2), x ** (1 / 2.0), x ** (1 / 2.4)], axis=1).astype(np.float32)
    return tstw, ctrl, wts, coefs.astype(np.float32), tmap


def cava_raw(batch=1, r=1080, c=1920, seed=0):
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, (min(batch, 4), 3, r, c), dtype=np.uint8)
    return np.stack([np.roll(base[f % len(base)], f // len(base), axis=2) for f in range(batch)])


# --------------------------------------------------------------------- SRAD
def srad_image(rows=16384, cols=16384, seed=0):
    """255 x smooth pattern x gamma speckle (ultrasound-like)."""
    rng = np.random.default_rng(seed)
    y = np.linspace(0, 4 * np.pi, rows, dtype=np.float32)[:, None]
    x = np.linspace(0, 4 * np.pi, cols, dtype=np.float32)[None, :]
    pattern = 0.55 + 0.35 * np.sin(y) * np.cos(x)
    speckle = rng.gamma(4.0, 0.25, (rows, cols)).astype(np.float32)
    return np.clip(255.0 * pattern * speckle / 2.0, 1.0, 255.0).astype(np.float32)


# ---------------------------------------------------------------- CFD/Euler
GAMMA = 1.4


def euler_ff_variable(mach=1.2, angle_deg=0.0):
    """Rodinia euler3d far-field state (density, momentum xyz, energy)."""
    rho = np.float32(1.4)
    p = np.float32(1.0)
    a = np.float32(np.sqrt(np.float32(GAMMA) * p / rho))
    sp = np.float32(mach) * a
    ang = np.float32(np.pi / 180.0 * angle_deg)
    v = np.array([sp * np.cos(ang), sp * np.sin(ang), 0.0], np.float32)
    mom = rho * v
    e = rho * (np.float32(0.5) * (sp * sp)) + p / np.float32(GAMMA - 1.0)
    return np.array([rho, mom[0], mom[1], mom[2], e], np.float32)


def euler_mesh(width=2048, height=2048, seed=0):
    """Structured-synthetic mesh: element (y,x) has neighbours W, E, S, N;
    top/bottom boundary faces are walls (-1), left/right far field (-2).
    Returns areas f32[nelr], neighbors i32[4,nelr], normals f32[4,3,nelr],
    ff_variable f32[5], variables f32[5,nelr] (far field + 1% perturbation)."""
    rng = np.random.default_rng(seed)
    nelr = width * height
    idx = np.arange(nelr, dtype=np.int64).reshape(height, width)
    nb = np.empty((4, height, width), np.int32)
    nb[0] = np.where(idx % width == 0, -2, idx - 1)
    nb[1] = np.where(idx % width == width - 1, -2, idx + 1)
    nb[2] = np.where(idx < width, -1, idx - width)
    nb[3] = np.where(idx >= (height - 1) * width, -1, idx + width)
    h = 1.0 / width
    base = np.array([[-h, 0, 0], [h, 0, 0], [0, -h, 0], [0, h, 0]], np.float32)
    normals = base[:, :, None] * (1.0 + 0.05 * rng.uniform(-1, 1, (4, 1, nelr)))
    normals[:, 2, :] = 0.01 * h * rng.uniform(-1, 1, (4, nelr))
    areas = (h * h * rng.uniform(0.5, 1.5, nelr)).astype(np.float32)
    ff = euler_ff_variable()
    variables = (ff[:, None] * (1.0 + 0.01 * rng.uniform(-1, 1, (5, nelr)))).astype(np.float32)
    return (areas, nb.reshape(4, nelr), normals.astype(np.float32), ff, variables)


# ---------------------------------------------------------------------- BFS
def bfs_graph(n=1 << 24, seed=42, max_degree=11):
    """Rodinia-style random graph in CSR: out-degree ~ U{1..max_degree},
    destinations uniform.  Returns starting, no_of_edges, edges (u32)."""
    rng = np.random.default_rng(seed)
    deg = rng.integers(1, max_degree + 1, n, dtype=np.uint32)
    starting = np.zeros(n, np.uint32)
    np.cumsum(deg[:-1], out=starting[1:])
    m = int(deg.sum(dtype=np.uint64))
    edges = rng.integers(0, n, m, dtype=np.uint32)
    return starting, deg, edges


# ----------------------------------------------------------------- backprop
def bp_inputs(n_in=1 << 24, n_hid=16, n_out=1, seed=7):
    """Rodinia backprop init: weights U[0,1), inputs U[0,1), prev weights 0,
    target 0.1 (bpnn_randomize_weights / load / bpnn_zero_weights)."""
    rng = np.random.default_rng(seed)
    x = rng.random(n_in + 1, dtype=np.float32)
    iw = rng.random((n_in + 1, n_hid + 1), dtype=np.float32)
    hw = rng.random((n_hid + 1, n_out + 1), dtype=np.float32)
    t = np.full(n_out + 1, 0.1, np.float32)
    ipw = np.zeros_like(iw)
    hpw = np.zeros_like(hw)
    return x, iw, hw, t, ipw, hpw


def bp_inputs_unsaturated(n_in=1 << 24, n_hid=16, n_out=1, seed=11):
    """A parity configuration where every stage is live: input weights
    U(-1,1)*4/sqrt(n_in) keep the hidden sums O(1) (Rodinia's U[0,1)
    weights drive them to ~4e6, where squash is exactly 1 and every delta
    and weight update is 0), and non-zero previous weights exercise the
    momentum term.  Inputs and target as Rodinia."""
    rng = np.random.default_rng(seed)
    x = rng.random(n_in + 1, dtype=np.float32)
    scale = np.float32(4.0 / np.sqrt(n_in))
    iw = ((rng.random((n_in + 1, n_hid + 1), dtype=np.float32) * np.float32(2) - np.float32(1)) * scale)
    hw = rng.random((n_hid + 1, n_out + 1), dtype=np.float32) * np.float32(2) - np.float32(1)
    t = np.full(n_out + 1, 0.1, np.float32)
    ipw = (rng.random(iw.shape, dtype=np.float32) - np.float32(0.5)) * np.float32(1e-3)
    hpw = (rng.random(hw.shape, dtype=np.float32) - np.float32(0.5)) * np.float32(1e-3)
    return x, iw.astype(np.float32), hw.astype(np.float32), t, ipw.astype(np.float32), hpw.astype(np.float32)
