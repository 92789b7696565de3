"""Pins for the oracle's w = 128 variant of Alg. 5 ("An initial block width of w=128 bits is
also possible and in this case the operative field is TGF(2^256)"; sec 4.2).

What pins what:
  * the end-to-end product against the plain definition (schoolbook / brute force, O1/O2);
  * TGF(2^256): field axioms, the defining relation x_8^2 + x_8 = v_127 (P:643-650 one level up),
    Frobenius: a^(2^256) = a for all a and x_8^(2^128) = x_8 + 1 (the top level is a field, not a
    split ring), the subfield embedding and Prop. 2;
  * GF(2^256) = GF(2)[z]/(z^256+z^10+z^5+z^2+1): Rabin's irreducibility test and the product against
    Python integer carry-less multiplication + reduction (R20);
  * changeRepr_256: the generators' defining relations, the smaller-root rule, ring homomorphism;
  * FFT_LCH over TGF(2^256) evaluates the polynomial at the tower points (Alg. 1 output order, R2).
"""
import random

import numpy as np
import pytest

import oracle as O
from oracle.brute import brute_mul_words, clmul_int
from gf2x_synth import operand, operand_pair, splitmix64

R = random.Random(1708)
P256 = (1 << 256) | (1 << 10) | (1 << 5) | (1 << 2) | 1


def rnd(bits):
    return R.getrandbits(bits)


# ---------------------------------------------------------------- GF(2^256), polynomial basis
def pmod(a, p):
    dp = p.bit_length() - 1
    while a and a.bit_length() - 1 >= dp:
        a ^= p << (a.bit_length() - 1 - dp)
    return a


def gf256p_ref(a, b):
    return pmod(clmul_int(a, b), P256)


def test_modulus_is_irreducible():
    # Rabin: p of degree 256 = 2^8 is irreducible iff z^(2^256) = z (mod p) and gcd(z^(2^128) - z, p) = 1
    def frob(k):
        y = 2
        for _ in range(k):
            y = gf256p_ref(y, y)
        return y

    def gcd(a, b):
        while b:
            a, b = b, pmod(a, b)
        return a

    assert frob(256) == 2
    assert gcd(frob(128) ^ 2, P256) == 1


def test_gf256p_mul_vs_definition():
    for _ in range(40):
        a, b = rnd(256), rnd(256)
        assert O.gf256p_mul(a, b) == gf256p_ref(a, b)


# ---------------------------------------------------------------- TGF(2^256)
def test_defining_relation_level8():
    x8, v127 = 1 << 128, 1 << 127
    assert O.tower256_mul(x8, x8) ^ x8 == v127


def test_field_axioms_sampled():
    for _ in range(40):
        a, b, c = rnd(256), rnd(256), rnd(256)
        ab = O.tower256_mul(a, b)
        assert ab == O.tower256_mul(b, a)
        assert O.tower256_mul(ab, c) == O.tower256_mul(a, O.tower256_mul(b, c))
        assert O.tower256_mul(a, b ^ c) == ab ^ O.tower256_mul(a, c)
        assert O.tower256_mul(a, 1) == a
        assert ab != 0


def test_frobenius_is_a_field_of_2_256():
    # every element is fixed by z -> z^(2^256); x_8 is not fixed by z -> z^(2^128) but sent to the
    # other root x_8 + 1 of x^2 + x + v_127 (so that polynomial is irreducible over TGF(2^128))
    def frob(x, k):
        for _ in range(k):
            x = O.tower256_mul(x, x)
        return x

    for a in [rnd(256) for _ in range(3)] + [1 << 128, (1 << 255) | 1]:
        assert frob(a, 256) == a
    assert frob(1 << 128, 128) == (1 << 128) ^ 1


def test_subfield_and_prop2():
    for _ in range(60):
        a, b = rnd(128), rnd(128)
        assert O.tower256_mul(a, b) == O.tower_mul(a, b)          # TGF(2^128) embedded in the low half
        A, c = rnd(256), rnd(32)
        lo, hi = A & ((1 << 128) - 1), A >> 128
        assert O.tower256_mul(A, c) == O.tower_mul(lo, c) | (O.tower_mul(hi, c) << 128)


# ---------------------------------------------------------------- changeRepr_256
def test_psi256_generators():
    prod = 1
    for k in range(1, 9):
        X = O.psi256_generator(k)
        assert gf256p_ref(X, X) ^ X == prod
        assert X < X ^ 1                      # the numerically smaller root (R9's rule)
        prod = gf256p_ref(prod, X)


def test_psi256_is_ring_isomorphism():
    assert O.psi256(1) == 1 and O.psi256_inv(1) == 1
    for _ in range(30):
        u, v = rnd(256), rnd(256)
        assert O.psi256(gf256p_ref(u, v)) == O.tower256_mul(O.psi256(u), O.psi256(v))
        assert O.psi256_inv(O.psi256(u)) == u
        assert O.psi256(u ^ v) == O.psi256(u) ^ O.psi256(v)


def test_psi256_low_degree_products_do_not_wrap():
    # the Kronecker argument of Alg. 5: blocks of degree < 128 multiply to degree <= 254 < 256, so
    # psi256^-1(psi256(a) psi256(b)) is the plain carry-less product
    for _ in range(30):
        a, b = rnd(128), rnd(128)
        assert O.psi256_inv(O.tower256_mul(O.psi256(a), O.psi256(b))) == clmul_int(a, b)


# ---------------------------------------------------------------- FFT_LCH over TGF(2^256)
def horner256(coeffs, alpha):
    acc = 0
    for c in reversed(coeffs):
        acc = O.tower256_mul(acc, alpha) ^ c
    return acc


@pytest.mark.parametrize("m", [1, 2, 3, 5])
def test_fft256_evaluates_at_tower_points(m):
    n = 1 << m
    coeffs = [rnd(256) for _ in range(n)]
    f = np.array([[(c >> (64 * i)) & (2**64 - 1) for i in range(4)] for c in coeffs], dtype=np.uint64)
    # BasisCvt is XOR-only on whole units: convert the low and high 128-bit halves
    g = np.concatenate([O.basis_cvt(f[:, 0:2].reshape(-1), 2).reshape(-1, 2),
                        O.basis_cvt(f[:, 2:4].reshape(-1), 2).reshape(-1, 2)], axis=1)
    e = O.fft256(g)
    for i in range(n):
        assert sum(int(e[i, j]) << (64 * j) for j in range(4)) == horner256(coeffs, i)


# ---------------------------------------------------------------- Alg. 5, w = 128, end to end
@pytest.mark.parametrize("bits", [1, 2, 64, 127, 128, 129, 255, 256, 257, 511, 512, 1000, 2048])
def test_alg5_w128_vs_brute(bits):
    a, b = operand_pair(bits, seed=bits + 3)
    assert np.array_equal(O.alg5_mul_w128(a, bits, b, bits), brute_mul_words(a, b))


def test_alg5_w128_unequal_ragged_and_large():
    for ab, bb in [(1, 1000), (128 * 7 + 3, 128 * 2), (5000, 130), (128, 128 * 64 + 1), (3, 2), (64, 65)]:
        a, b = operand(ab, seed=ab), operand(bb, seed=bb + 1)
        assert np.array_equal(O.alg5_mul_w128(a, ab, b, bb), brute_mul_words(a, b))
    for bits in [1 << 16, (1 << 16) + 77]:
        a, b = operand_pair(bits, seed=9)
        assert np.array_equal(O.alg5_mul_w128(a, bits, b, bits), O.mul_schoolbook(a, b))


def test_alg5_w128_edge_cases():
    a = operand(300, seed=4)
    assert not O.alg5_mul_w128(a, 300, np.zeros(1, np.uint64), 0).any()
    one = np.array([1], dtype=np.uint64)
    c = O.alg5_mul_w128(a, 300, one, 1)
    assert np.array_equal(c[:len(a)], a) and not c[len(a):].any()
    # bits of the operands above a_bits are ignored
    noisy = a.copy()
    noisy[-1] |= np.uint64(0xFFFF) << np.uint64(50)
    assert np.array_equal(O.alg5_mul_w128(noisy, 300, a, 300), O.alg5_mul_w128(a, 300, a, 300))


def test_alg5_w128_stages():
    bits = 4096
    a, b = operand_pair(bits, seed=21)
    c, st = O.alg5_mul_w128(a, bits, b, bits, stages=True)
    N = len(st["cvt_a"])
    assert N == 64
    # after changeRepr the upper half of the points is zero (degree < 32 blocks, Kronecker padding)
    assert not st["cvt_a"][32:].any()
    # FFT output = FFT of the changeRepr stage
    assert np.array_equal(O.fft256(st["cvt_a"]), st["fft_a"])
    assert np.array_equal(c, brute_mul_words(a, b))
