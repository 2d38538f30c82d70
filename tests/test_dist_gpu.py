"""Row-slab SRAD building blocks on the GPU: the slab kernels driven by the
dist.py host logic (world 1), and a 3-slab decomposition emulated in one
process (device-side halo copies) -- both bit-identical to the oracle."""
import numpy as np
import pytest

from paper_2503_10855_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_srad_distributed_world1_matches_oracle(jb, oracle):
    import torch
    from paper_2503_10855_b200 import dist as D
    img = W.srad_image(96, 130, seed=2)
    out = D.srad_distributed(torch.from_numpy(img).cuda(), 5, 0.5, 96, 130, D.CudaSradBackend()).cpu().numpy()
    ref = oracle.srad(img, 5, 0.5)
    assert np.count_nonzero(out.view(np.uint32) != ref.view(np.uint32)) <= out.size // 10000
    np.testing.assert_allclose(out, ref, rtol=1e-5)


@pytest.mark.parametrize("nslab", [2, 3])
def test_srad_emulated_slabs_match_oracle(jb, oracle, nslab):
    import torch
    from paper_2503_10855_b200 import dist as D
    rows, cols, niter = 70, 150, 4
    img = W.srad_image(rows, cols, seed=4)
    be = D.CudaSradBackend()
    plans = [D.srad_slab(rows, nslab, r) for r in range(nslab)]
    Js, sums = [], []
    for p in plans:
        J, s = be.extract(torch.from_numpy(np.ascontiguousarray(img[p["r0"]:p["r1"]])).cuda(), False)
        Js.append(J)
        sums.append(s)
    q0 = be.q0(sum(sums), rows * cols)
    for it in range(niter):
        last = it + 1 == niter
        full = torch.cat(Js, 0)  # the halo exchange, done with one device copy
        new, sums = [], []
        for p in plans:
            o, s = be.step(full[p["e0"]:p["e1"]].contiguous(), p["own_lo"], p["own_hi"], q0, 0.5, last)
            new.append(o)
            sums.append(s)
        Js = new
        if not last:
            q0 = be.q0(sum(sums), rows * cols)
    got = torch.cat(Js, 0).cpu().numpy()
    ref = oracle.srad(img, niter, 0.5)
    assert np.count_nonzero(got.view(np.uint32) != ref.view(np.uint32)) <= got.size // 10000
    np.testing.assert_allclose(got, ref, rtol=1e-5)
