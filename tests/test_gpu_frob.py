"""GPU parity of App. C's first step: BasisCvt / iBasisCvt on GF(2) coefficients
(gf2x_basis_cvt_bits) against the oracle's bit-level Alg. 3 (O.basis_cvt_bits, pinned in test_oracle_frob.py).
Bit-exact; the full App. C multiply on the GPU is the next step."""
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


@pytest.mark.parametrize("M", [6, 7, 8, 9, 11, 12, 16, 17, 20, 23])
def test_bit_basis_cvt_matches_oracle(M):
    f = operand(1 << M, seed=M + 500)
    d = dev(f)
    G.gf2x_basis_cvt_bits(d, M)
    g = host(d)
    assert np.array_equal(g, O.basis_cvt_bits(f, M))
    G.gf2x_basis_cvt_bits(d, M, inverse=True)
    assert np.array_equal(host(d), f)
    d2 = dev(g)
    G.gf2x_basis_cvt_bits(d2, M, inverse=True)
    assert np.array_equal(host(d2), O.basis_cvt_bits(g, M, inverse=True))


def test_bit_basis_cvt_sparse_and_edge_inputs():
    M = 10
    for f in [np.zeros(1 << (M - 6), np.uint64), np.full(1 << (M - 6), np.uint64(0xFFFFFFFFFFFFFFFF))]:
        d = dev(f)
        G.gf2x_basis_cvt_bits(d, M)
        assert np.array_equal(host(d), O.basis_cvt_bits(f, M))
    for t in [0, 1, 63, 64, 511, 512, 1023]:   # monomials x^t
        f = np.zeros(1 << (M - 6), np.uint64)
        f[t // 64] = np.uint64(1 << (t % 64))
        d = dev(f)
        G.gf2x_basis_cvt_bits(d, M)
        assert np.array_equal(host(d), O.basis_cvt_bits(f, M)), t
    with pytest.raises(G.Gf2xError):
        G.gf2x_basis_cvt_bits(dev(np.zeros(1, np.uint64)), 5)


def test_bit_basis_cvt_full_size_roundtrip():
    # the size the App. C multiply of two 2^29-bit operands converts (2^30 coefficients): the inverse returns
    # the input, and sampled words of a sparse input match the oracle at a size it converts in seconds
    M = 30
    f = operand(1 << M, seed=77)
    d = dev(f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.gf2x_basis_cvt_bits(d, M)
    e1.record()
    torch.cuda.synchronize()
    print(f"bit-level BasisCvt, 2^{M} coefficients: {e0.elapsed_time(e1):.2f} ms")
    G.gf2x_basis_cvt_bits(d, M, inverse=True)
    assert np.array_equal(host(d), f)
