"""Pins for the oracle's App. C multiply through the Frobenius bijection (
DESIGN.md R23).

What pins what:
  * the end-to-end product against brute-force carry-less multiplication (any mistake in BasisCvt on
    bits, the encoding, the alpha-displaced FFT, decoding or iBasisCvt breaks it);
  * E(a)_i = a(beta_(m+64) + phi(i)) by Horner over the tower (Def. P:1502-1507) -- the forward half
    against the plain definition, independent of the FFT and of BasisCvt;
  * the encoding's columns against the paper's closed form prod_{bit k of j} s_(m+7-k)(beta_(m+64))
     and their rank 128 (the bijection, Prop. P:1515-1518);
  * the Frobenius order of beta_(m+64) is 128.
"""
import random

import numpy as np
import pytest

import oracle as O
from oracle.brute import brute_mul_words
from gf2x_synth import operand

R = random.Random(1485)


def horner_bits(a, a_bits, x):
    acc = 0
    for t in reversed(range(a_bits)):
        acc = O.tower_mul(acc, x) ^ ((int(a[t // 64]) >> (t % 64)) & 1)
    return acc


def rank_gf2(vectors):
    basis = {}
    for v in vectors:
        while v:
            h = v.bit_length() - 1
            if h not in basis:
                basis[h] = v
                break
            v ^= basis[h]
    return len(basis)


@pytest.mark.parametrize("bits", [1, 2, 63, 64, 65, 127, 128, 129, 255, 256, 257, 511, 512, 513, 1000, 2048, 4097, 8191])
def test_frob_mul_square_sizes(bits):
    a, b = operand(bits, seed=bits + 40), operand(bits, seed=bits + 41)
    assert np.array_equal(O.frob_mul(a, bits, b, bits), brute_mul_words(a, b))


@pytest.mark.parametrize("ab,bb", [(1, 1000), (1000, 1), (64, 65), (128, 129), (300, 4000), (128 * 16, 128 * 16 + 1),
                                   (3, 2), (5000, 130)])
def test_frob_mul_unequal_sizes(ab, bb):
    a, b = operand(ab, seed=ab), operand(bb, seed=bb + 7)
    c = O.frob_mul(a, ab, b, bb)
    assert np.array_equal(c, brute_mul_words(a, b))
    assert np.array_equal(O.frob_mul(b, bb, a, ab), c)


def test_frob_mul_point_count_boundaries():
    # L = a_bits + b_bits - 1 coefficients need 128 * 2^m >= L points' worth of bits (R23)
    assert O.frob_m(64, 65) == 0 and O.frob_m(65, 65) == 1
    assert O.frob_m(1024, 1025) == 4 and O.frob_m(1025, 1025) == 5
    for ab, bb in [(64, 65), (65, 65), (1024, 1025), (1025, 1025)]:
        a, b = operand(ab, seed=1), operand(bb, seed=2)
        assert np.array_equal(O.frob_mul(a, ab, b, bb), brute_mul_words(a, b))


def test_frob_mul_edge_cases():
    a = operand(700, seed=3)
    assert not O.frob_mul(a, 700, np.zeros(1, np.uint64), 0).any()
    one = np.array([1], dtype=np.uint64)
    c = O.frob_mul(a, 700, one, 1)
    assert np.array_equal(c[:len(a)], a) and not c[len(a):].any()
    noisy = a.copy()
    noisy[-1] |= np.uint64(0xF) << np.uint64(60)   # bits 700.. (above a_bits) are ignored
    assert np.array_equal(O.frob_mul(noisy, 700, a, 700), O.frob_mul(a, 700, a, 700))


@pytest.mark.parametrize("m,bits", [(0, 128), (0, 77), (1, 256), (2, 512), (2, 300), (3, 1024)])
def test_frob_eval_is_evaluation_at_the_shifted_points(m, bits):
    a = operand(bits, seed=m * 100 + bits)
    E = O.frob_eval(a, bits, m)
    alpha = 1 << (m + 64)
    for i in range(1 << m):
        got = int(E[i, 0]) | (int(E[i, 1]) << 64)
        assert got == horner_bits(a, bits, alpha ^ i), i


@pytest.mark.parametrize("m", [0, 1, 4, 10, 20])
def test_encoding_columns_closed_form_and_rank(m):
    # column j = prod_{k-th bit of j is 1} s_(m+7-k)(beta_(m+64)), reading the bits of j from the
    # most significant (k = 1 .. 7), i.e. bit b (LSB = 0) carries s_(m+b) (R23)
    alpha = 1 << (m + 64)
    s = {b: O.s_eval(m + b, alpha) for b in range(7)}
    cols = O.frob_columns(m)
    for j in range(128):
        c = 1
        for k in range(1, 8):
            if (j >> (7 - k)) & 1:
                c = O.tower_mul(c, O.s_eval(m + 7 - k, alpha))
        assert cols[j] == c, j
        c2 = 1
        for b in range(7):
            if (j >> b) & 1:
                c2 = O.tower_mul(c2, s[b])
        assert c2 == c
    assert rank_gf2(cols) == 128


@pytest.mark.parametrize("m", [0, 1])
def test_bijection_on_monomials(m):
    # Prop. P:1515-1518: E is a bijection GF(2)[x]_{<128 n} -> GF(2^128)^n; it is linear, so the images of the
    # 128 n monomials must be independent (n = 1: a(alpha) determines a of degree < 128)
    n = 1 << m
    vecs = []
    for t in range(128 * n):
        a = np.zeros((t + 64) // 64, dtype=np.uint64)
        a[t // 64] = np.uint64(1 << (t % 64))
        E = O.frob_eval(a, t + 1, m)
        v = 0
        for i in range(n):
            v |= (int(E[i, 0]) | (int(E[i, 1]) << 64)) << (128 * i)
        vecs.append(v)
    assert rank_gf2(vecs) == 128 * n


@pytest.mark.parametrize("m", [0, 5, 17, 40])
def test_frobenius_order_of_alpha(m):
    # the order of phi_2 on beta_(m+64) is 128 (2 * 2^floor(log2(m+64)))
    alpha = 1 << (m + 64)
    x = alpha
    for i in range(1, 129):
        x = O.tower_mul(x, x)
        if i == 64:
            assert x != alpha
    assert x == alpha


@pytest.mark.parametrize("M", [6, 7, 9])
def test_bit_level_basis_cvt_is_the_novel_basis_expansion(M):
    # f(alpha) = sum_i g_i X_i(alpha) with X_i = prod_{bit k of i} s_k (Cantor-normalised novel basis),
    # at random tower points alpha; and the inverse returns f
    f = operand(1 << M, seed=M)
    g = O.basis_cvt_bits(f, M)
    assert np.array_equal(O.basis_cvt_bits(g, M, inverse=True), f)
    for t in range(3):
        alpha = R.getrandbits(128)
        s = [O.s_eval(k, alpha) for k in range(M)]
        acc = 0
        for i in range(1 << M):
            if (int(g[i // 64]) >> (i % 64)) & 1:
                x = 1
                for k in range(M):
                    if (i >> k) & 1:
                        x = O.tower_mul(x, s[k])
                acc ^= x
        assert acc == horner_bits(f, 1 << M, alpha), t
