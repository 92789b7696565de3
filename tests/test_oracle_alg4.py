"""Pins for the oracle's Alg. 4 (sec 3.1: FFT_LCH directly in GF(2^128), polynomial basis, with the
multipliers s_k computed in the Cantor/tower basis and mapped by the field isomorphism).

  * the product against brute force (the plain definition);
  * FFT_LCH over GF(2^128) evaluates the polynomial at the points psi^-1(phi_v(i)) (Horner, gf128);
  * conjugation: Alg. 4's transform is psi^-1 o (the tower FFT) o psi element-wise, since psi is a field
    isomorphism (pinned independently in test_oracle_tower.py).
"""
import random

import numpy as np
import pytest

import oracle as O
from oracle.brute import brute_mul_words
from gf2x_synth import operand, operand_pair, splitmix64

R = random.Random(404)


@pytest.mark.parametrize("bits", [1, 2, 63, 64, 65, 127, 128, 129, 511, 512, 513, 2048, 4097])
def test_alg4_vs_brute(bits):
    a, b = operand_pair(bits, seed=bits + 40)
    assert np.array_equal(O.alg4_mul(a, bits, b, bits), brute_mul_words(a, b))


def test_alg4_unequal_ragged_and_large():
    for ab, bb in [(1, 1000), (64 * 7 + 3, 128), (5000, 130), (3, 2)]:
        a, b = operand(ab, seed=ab + 1), operand(bb, seed=bb + 2)
        assert np.array_equal(O.alg4_mul(a, ab, b, bb), brute_mul_words(a, b))
    bits = 1 << 16
    a, b = operand_pair(bits, seed=12)
    assert np.array_equal(O.alg4_mul(a, bits, b, bits), O.mul_karatsuba(a, b))


def horner_gf128(coeffs, x):
    acc = 0
    for c in reversed(coeffs):
        acc = O.gf128_mul(acc, x) ^ c
    return acc


@pytest.mark.parametrize("m", [1, 2, 3, 5])
def test_fft_alg4_evaluates_at_mapped_points(m):
    n = 1 << m
    coeffs = [R.getrandbits(128) for _ in range(n)]
    f = np.array([[c & (2**64 - 1), c >> 64] for c in coeffs], dtype=np.uint64)
    g = O.basis_cvt(f.reshape(-1), 2).reshape(-1, 2)
    e = O.fft_alg4(g)
    for i in range(n):
        assert int(e[i, 0]) | (int(e[i, 1]) << 64) == horner_gf128(coeffs, O.psi_inv(i))


@pytest.mark.parametrize("m", [4, 9])
def test_fft_alg4_is_conjugate_of_tower_fft(m):
    g = splitmix64(77 + m, 2 << m).reshape(-1, 2)
    to_int = lambda r: int(r[0]) | (int(r[1]) << 64)
    to_row = lambda v: [v & (2**64 - 1), v >> 64]
    gt = np.array([to_row(O.psi(to_int(r))) for r in g], dtype=np.uint64)
    et = O.fft(gt)
    want = np.array([to_row(O.psi_inv(to_int(r))) for r in et], dtype=np.uint64)
    assert np.array_equal(O.fft_alg4(g), want)
