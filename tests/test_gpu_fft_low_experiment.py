"""The warp-shuffle experiment of DESIGN.md §7 (not on the product path): the five innermost forward FFT
layers as one element per lane with shuffles (gf2x_experiment_fft_low variant 1) equal k_bottom's bit-sliced
layers (variant 0, the product path's formulation, itself pinned by the stage parity tests against the
oracle's Alg. 1) on the same seeded spectra."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import splitmix64  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1708_09746_b200 import build
    build.build()
    G.load()


@pytest.mark.parametrize("m", [11, 14, 20])
def test_shuffle_layers_equal_bitsliced(m):
    n = 1 << m
    w = splitmix64(321 + m, 4 * n).reshape(2, n, 2)
    A0 = torch.from_numpy(w[0].view(np.int64).copy()).cuda().view(torch.uint64)
    B0 = torch.from_numpy(w[1].view(np.int64).copy()).cuda().view(torch.uint64)
    A1, B1 = A0.clone(), B0.clone()
    G.experiment_fft_low(A0, B0, m, 0)
    G.experiment_fft_low(A1, B1, m, 1)
    torch.cuda.synchronize()
    assert torch.equal(A0, A1) and torch.equal(B0, B1)
    assert not torch.equal(A0, torch.from_numpy(w[0].view(np.int64).copy()).cuda().view(torch.uint64))
