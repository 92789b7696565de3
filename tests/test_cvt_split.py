"""Pins for DESIGN.md R22: BasisCvt / iBasisCvt of a polynomial whose length is just above a power of
two split into a conversion of the lower half and a small one of the tail (used by the GPU path for
ragged operands and truncated products).  Checked against the oracle's full-size Alg. 3 (O3), which is
itself pinned to the novel basis in test_oracle_transforms.py.

With X_(2^p) = s_p(x) (the tower basis is Cantor's, s_p(v_p) = 1) and s_p = sum_{q subset of p} x^(2^q)
(Lucas, P:327 recursion; test_oracle_tower.s_exponents):
  forward:  f = f_lo + x^(2^p) f_hi, deg f_hi < 2^j  ==>
            BasisCvt_(p+1)(f) = [BasisCvt_p(f_lo + sum_{q subset p, q != p} x^(2^q) f_hi), BasisCvt_j(f_hi), 0...]
  inverse:  g = [g_lo (2^p), g_hi (2^j), 0...]  ==>
            iBasisCvt_(p+1)(g) = iBasisCvt_p(g_lo) + s_p(x) * iBasisCvt_j(g_hi)
"""
import numpy as np
import pytest

import oracle as O
from gf2x_synth import splitmix64


def s_exponents(i):
    s = {0}
    for _ in range(i):
        s = {j + 1 for j in s} ^ s
    return s


def rand_words(n, seed):
    return splitmix64(seed, n)


def ceil_log2(x):
    return max(0, (x - 1).bit_length())


@pytest.mark.parametrize("p,r", [(6, 1), (7, 3), (8, 16), (9, 17), (10, 1), (11, 100), (12, 256), (13, 1000)])
def test_forward_split(p, r):
    w = 1
    f = np.zeros(2 << p, dtype=np.uint64)
    f[:(1 << p) + r] = rand_words((1 << p) + r, seed=p * 31 + r)
    full = O.basis_cvt(f, w)
    j = ceil_log2(r)
    lo = f[:1 << p].copy()
    hi = f[1 << p:(1 << p) + (1 << j)].copy()
    for q in s_exponents(p) - {p}:
        assert (1 << q) + (1 << j) <= 1 << p
        lo[1 << q:(1 << q) + (1 << j)] ^= hi
    got = np.zeros_like(f)
    got[:1 << p] = O.basis_cvt(lo, w)
    got[1 << p:(1 << p) + (1 << j)] = O.basis_cvt(hi, w) if j else hi
    assert np.array_equal(got, full)


@pytest.mark.parametrize("p,j", [(6, 0), (7, 2), (8, 4), (9, 5), (10, 8), (11, 9), (12, 10)])
def test_inverse_split(p, j):
    w = 2   # 128-bit units, as the product side
    g = np.zeros((2 << p) * w, dtype=np.uint64)
    g[:((1 << p) + (1 << j)) * w] = rand_words(((1 << p) + (1 << j)) * w, seed=p * 17 + j)
    full = O.ibasis_cvt(g, w).reshape(-1, w)
    lo = O.ibasis_cvt(g[:(1 << p) * w], w).reshape(-1, w)
    hi = g[(1 << p) * w:((1 << p) + (1 << j)) * w]
    q = (O.ibasis_cvt(hi, w) if j else hi).reshape(-1, w)
    got = np.zeros_like(full)
    got[:1 << p] = lo
    for e in s_exponents(p):
        got[1 << e:(1 << e) + (1 << j)] ^= q
    assert np.array_equal(got, full)


def test_split_needs_the_lucas_terms():
    # dropping the x^(2^q) fold-in (q != p) breaks the identity: the fold is what the split is about
    p, r = 9, 40
    f = np.zeros(2 << p, dtype=np.uint64)
    f[:(1 << p) + r] = rand_words((1 << p) + r, seed=5)
    j = ceil_log2(r)
    got = np.zeros_like(f)
    got[:1 << p] = O.basis_cvt(f[:1 << p], 1)
    got[1 << p:(1 << p) + (1 << j)] = O.basis_cvt(f[1 << p:(1 << p) + (1 << j)], 1)
    assert not np.array_equal(got, O.basis_cvt(f, 1))
