"""CAVA camera pipeline on the B200 vs the oracle restatement: bit-exact u8."""
import numpy as np
import pytest

from conftest import golden
from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,P", [((1, 64, 96), 16), ((2, 33, 70), 16), ((1, 135, 240), 64),
                                     ((1, 3, 3), 4), ((1, 1080, 1920), 16), ((3, 70, 130), 0)])
def test_cava_matches_oracle(jb, oracle, shape, P):
    b, r, c = shape
    raw = W.cava_raw(b, r, c, seed=r)
    params = W.cava_params(P=max(P, 1))
    if P == 0:
        params = (params[0], params[1][:0], params[2][:0], params[3], params[4])
    got = jb.cava(raw, *params)
    ref = oracle.cava(raw, *params)
    assert got.dtype == np.uint8 and got.shape == raw.shape
    bad = np.count_nonzero(got != ref)
    assert bad == 0, f"{bad}/{got.size} u8 values differ (max |d| {np.abs(got.astype(int) - ref).max()})"


@pytest.mark.parametrize("P", [63, 64, 255, 256, 257, 1024, 4096])
def test_cava_many_control_points(jb, oracle, P):
    """Control-point counts either side of the shared-memory table limit
    (PMAX_SMEM = 256 in cava.cu; larger tables stream from global memory)
    up to the compute variant's thousands of points, and either side of the
    switch to the fma(d, w, +0) weight products (CAVA_FMA0_MIN_P = 64)."""
    raw = W.cava_raw(2, 40, 72, seed=P)
    params = W.cava_params(P=P, seed=P)
    got = jb.cava(raw, *params)
    ref = oracle.cava(raw, *params)
    bad = np.count_nonzero(got != ref)
    assert bad == 0, f"P={P}: {bad}/{got.size} u8 values differ"


def test_cava_scale_transform_pinned(oracle):
    g = golden("cava_stages_6x8")
    sc = oracle.cava_stage("scale", g["raw"])
    assert np.array_equal(sc.view(np.uint32), g["scaled"].view(np.uint32))


def test_cava_pipelined_matches_single_call(jb):
    """The host-buffer pipelined entry (chunks through two device slots on
    three streams) returns exactly the single-call result, including a
    ragged last chunk."""
    import torch
    from paper_2503_10855_b200 import api
    raw = W.cava_raw(5, 70, 132, seed=3)
    params = W.cava_params(P=16)
    ref = jb.cava(raw, *params)
    got = api.cava_pipelined(torch.from_numpy(raw).pin_memory(), *params, chunk=2)
    assert np.array_equal(got.numpy(), ref)
