"""GPU parity of the split BasisCvt / iBasisCvt (R22; pinned on the CPU in test_cvt_split.py):
one product whose operand or result length is just above a power of two converts the lower half and the
short tail separately (k_shift_xor adds the s_p(x) shift terms).  Exact against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import operand  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def gpu_mul(a, ab, b, bb):
    G.profile_enable(True)
    c = host(G.gf2x_mul(dev(a), ab, dev(b), bb))
    names = {r["kernel"] for r in G.profile_report()}
    G.profile_enable(False)
    return c, names


W = 64
CASES = [
    # (a words, b words, split expected): full path (n_a > H), the tail of a and of the result split
    ((1 << 16) + 5, 3, True),
    ((1 << 17) + 5, (1 << 16) + 3, True),
    # tail exactly a quarter (j = p - 2, the largest split) and just above it (no split of a)
    ((1 << 16) + (1 << 14), 2, True),
    ((1 << 16) + (1 << 14) + 1, 1, False),
    # a truncated-FFT product (both operands and the result split); both operands split on the full path
    ((1 << 16) + 1, (1 << 16) + 1, True),
    ((1 << 18) + 77, (1 << 17) + 4000, True),
    # below the size threshold: not split
    ((1 << 13) + 1, (1 << 13) + 1, False),
]


@pytest.mark.parametrize("na,nb,split", CASES)
def test_split_products_exact(na, nb, split):
    ab, bb = na * W - 17, nb * W - 3
    a, b = operand(ab, seed=na % 977), operand(bb, seed=nb % 991 + 1)
    got, names = gpu_mul(a, ab, b, bb)
    assert ("k_shift_xor" in names) == split
    n = max(len(a), len(b))
    ref = O.mul_karatsuba(np.pad(a, (0, n - len(a))), np.pad(b, (0, n - len(b))))
    assert not ref[len(a) + len(b):].any()
    assert np.array_equal(got, ref[:len(a) + len(b)])
    got2, _ = gpu_mul(b, bb, a, ab)
    assert np.array_equal(got2, got)


def test_plan_reports_split():
    p = G.gf2x_plan(((1 << 16) + 5) * W, 3 * W)
    assert p["split"]["a"] == [16, 3] and p["split"]["b"] is None and p["split"]["icvt"] == [16, 3]
