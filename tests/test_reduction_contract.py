"""The global float reductions' contract (DESIGN.md §Reduction policy).

SRAD's Σ/Σ² and backprop's layer sums are ``monoid_reduce`` folds that the
paper's schedules re-associate (passes/monoid.py:21-31).  The
GPU kernels accumulate them in f64 and round once; the reference interpreter
folds them sequentially in f32 (oracle.py:288-304).  These CPU tests pin the
contract side (the f64 result is the correctly rounded exact sum) and bound
the distance to the reference fold with the textbook error analysis.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2503_10855_b200 import workloads as W

U = 2.0 ** -24


def _gamma(n):
    return n * U / (1 - n * U)


def test_srad_q0_f64_is_the_rounded_exact_value():
    img = W.srad_image(256, 256)
    _, q64 = O.srad(img, 1, 0.5, return_q0=True)
    J = O.srad_extract(img).astype(np.float64).ravel()   # the oracle's own J = exp_ref(I/255)
    s, s2 = math.fsum(J), math.fsum(J * J)
    mean = s / J.size
    q_exact = (s2 / J.size - mean * mean) / (mean * mean)
    assert abs(float(q64[0]) - q_exact) <= 2 * U * q_exact


def test_srad_f32_fold_within_its_error_bound_at_small_size():
    """The reference's sequential f32 fold against the f64 contract: within
    the propagated gamma_N bound of the two sums at 512^2 (q0 amplifies the
    sums' error by (E[J^2] + 2 mean^2) / var through the cancellation)."""
    img = W.srad_image(512, 512)
    _, q64 = O.srad(img, 1, 0.5, return_q0=True)
    _, q32 = O.srad(img, 1, 0.5, return_q0=True, acc64=False)
    q = float(q64[0])
    g = _gamma(512 * 512) + 2 * U
    amp = (1 + q) / q + 2 / q          # E2/var + 2 mean^2/var, in units of mean^2
    bound = (amp + 2) * g * q
    assert abs(float(q32[0]) - q) <= bound
    assert float(q32[0]) != q          # the two folds do differ


def test_srad_f32_fold_breaks_down_at_scale():
    """Why the contract is f64: at 4096^2 (2^24 pixels, sums ~3e7 > 2^24) the
    sequential f32 fold has lost the variance (DESIGN.md gives 16384^2:
    q0^2 = 7.45 against 0.0352)."""
    img = W.srad_image(4096, 4096)
    _, q64 = O.srad(img, 1, 0.5, return_q0=True)
    _, q32 = O.srad(img, 1, 0.5, return_q0=True, acc64=False)
    assert abs(float(q32[0]) - float(q64[0])) > 0.1 * float(q64[0])


@pytest.mark.parametrize("n", [1000, 65536])
def test_backprop_layer_sums_f64_vs_sequential_fold(n):
    x, iw, *_ = W.bp_inputs_unsaturated(n, 16, 1, seed=n)
    xs = x.copy()
    xs[0] = 1.0
    seq = O.bp_layer_sums(xs, iw, acc64=False)
    s64 = O.bp_layer_sums(xs, iw, acc64=True)
    prods = iw.astype(np.float32) * xs[:, None]          # the f32 products both folds add
    exact = np.array([math.fsum(prods[:, j].astype(np.float64)) for j in range(iw.shape[1])])
    abs_sum = np.abs(prods.astype(np.float64)).sum(axis=0)
    # f64 contract: the rounded exact sum (f64 accumulation error << u)
    assert np.all(np.abs(s64.astype(np.float64) - exact) <= U * np.abs(exact) + 1e-12 * abs_sum)
    # reference fold: Higham Thm 4.4, gamma_{n} * sum|x_i| (n*u < 1 here)
    assert np.all(np.abs(seq.astype(np.float64) - exact) <= _gamma(n + 1) * abs_sum)
