"""The branch-free division / reciprocal / sqrt sequences (csrc/common.cuh)
that the SRAD, CFD and CAVA kernels run inside their range guards must be
bit-identical to IEEE __fdiv_rn / __fsqrt_rn there."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lo,hi,seed", [(-60, 60, 1), (-96, 96, 2), (-8, 8, 3), (-1, 1, 4)])
def test_fast_paths_match_ieee(jb, lo, hi, seed):
    import torch
    from paper_2503_10855_b200 import _lib
    bad = torch.zeros(4, dtype=torch.int64, device="cuda")
    n = 1 << 27
    st = _lib.load().jb_selftest_fastmath(n, seed, lo, hi, bad.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream)
    assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert bad.tolist() == [0, 0, 0, 0], f"div/rcp/sqrt/div_by mismatches over {n} pairs: {bad.tolist()}"
