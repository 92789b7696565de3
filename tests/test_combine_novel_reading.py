"""Host-side pin of DESIGN.md R28, which k_ipsi_bs<true> + the 64-bit iBasisCvt rely on (gf2x.cu): Alg. 5's last
two steps (iBasisCvt P:901, changeRepr^-1 P:902, InterleavedCombine P:903: out[w] = lo64(C_w) ^ hi64(C_(w-1)))
equal iBasisCvt, on 64-bit words, of
    D = lo64(G) ^ M hi64(G),   (M h)[j] = h[j-1] ^ [j odd] h[j] ^ [j even, j > 0] h[j + 2^ctz(j) - 1],
G = changeRepr^-1 of the iFFT output (novel-basis coefficients).  M is the shift by one block (multiplication by
y = X_1 = s_0) written in the novel basis: X_1 X_k = X_(k+1) for even k, and for odd k the carries of s_j^2 =
s_(j+1) + s_j (s_(i+1) = s_1 o s_i) add X_k and X_(k+1-2^i), 1 <= i < trailing ones of k.
Checked against the oracle's own iBasisCvt and its full Alg. 5 (stages), so a wrong term or index fails."""
import numpy as np
import pytest

import oracle as O
from gf2x_synth import operand_pair


def m_shift(h):
    N = len(h)
    out = np.zeros_like(h)
    out[1:] ^= h[:-1]
    j = np.arange(N)
    odd = (j & 1) == 1
    out[odd] ^= h[odd]
    ev = np.nonzero(((j & 1) == 0) & (j > 0))[0]
    out[ev] ^= h[ev + (ev & -ev) - 1]
    return out


@pytest.mark.parametrize("m", [1, 2, 5, 9, 14])
def test_shift_in_novel_basis(m):
    N = 1 << m
    h = np.random.default_rng(m).integers(0, 1 << 63, size=N, dtype=np.uint64)
    h[-1] = 0   # the top coefficient of hi64 is zero for every product (degree bound)
    th = O.ibasis_cvt(h, 1)
    shifted = np.zeros_like(th)
    shifted[1:] = th[:-1]
    assert th[-1] == 0
    assert np.array_equal(O.ibasis_cvt(m_shift(h), 1), shifted)


@pytest.mark.parametrize("bits", [1 << 9, 1 << 12, 1 << 15, 3 << 12])
def test_product_through_novel_combine(bits):
    a, b = operand_pair(bits)
    c, st = O.alg5_mul(a, bits, b, bits, stages=True)
    G = st["ifft"]                                   # tower-basis novel coefficients after iFFT_LCH, (N, 2)
    N = 1 << ((2 * ((bits + 63) // 64) - 1) - 1).bit_length()
    G = G[:N]
    lo = np.zeros(N, dtype=np.uint64)
    hi = np.zeros(N, dtype=np.uint64)
    for k in range(N):
        v = O.psi_inv(int(G[k, 0]) | (int(G[k, 1]) << 64))
        lo[k] = v & ((1 << 64) - 1)
        hi[k] = v >> 64
    assert hi[-1] == 0
    got = O.ibasis_cvt(lo ^ m_shift(hi), 1)
    n_out = len(c)
    assert np.array_equal(got[:n_out], c)
    assert not np.any(got[n_out:])
