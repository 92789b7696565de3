"""The tensor-core experiment of DESIGN.md §7 (not on the product path): changeRepr^-1 as a tcgen05.mma kind::i8
product of 0/1 bytes with the accumulator in TMEM (gf2x_experiment_ipsi_tc) equals the oracle's psi^-1 (the same
isomorphism rule R9) element by element, including a ragged last tile."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import splitmix64  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1708_09746_b200 import build
    build.build()
    G.load()


@pytest.mark.parametrize("n", [128, 4096 + 77])
def test_ipsi_tc_matches_oracle(n):
    w = splitmix64(12345 + n, 2 * n).reshape(n, 2)
    w[:, 1] &= np.uint64((1 << 63) - 1)   # (any 128-bit value; keep one bit clear for variety)
    P = torch.from_numpy(w.view(np.int64).copy()).cuda().view(torch.uint64)
    out = G.experiment_ipsi_tc(P)
    torch.cuda.synchronize()
    got = out.cpu().view(torch.int64).numpy().view(np.uint64)
    rng = np.random.default_rng(n)
    idx = sorted(set([0, 1, 127, n - 1] + [int(x) for x in rng.integers(0, n, size=60)]))
    for i in idx:
        want = O.psi_inv(int(w[i, 0]) | (int(w[i, 1]) << 64))
        assert (int(got[i, 0]) | (int(got[i, 1]) << 64)) == want, i
