"""Pins for oracle O3 transforms: BasisCvt / iBasisCvt (Alg. 2/3 P:492-539, App. B),
FFT_LCH / iFFT (Alg. 1) and the full Alg. 5 pipeline."""
import random

import numpy as np
import pytest

import oracle as O
from oracle.brute import brute_mul_words, clmul_int, square_closed_form, shift_closed_form
from gf2x_synth import operand, operand_pair, splitmix64
from tests.test_oracle_tower import s_symbolic

R = random.Random(5)


def X_poly(k):
    """novel-poly basis X_k(x) = prod_{bit i of k} s_i(x) in GF(2)[x] (Def. 3)."""
    p = 1
    i = 0
    while k >> i:
        if (k >> i) & 1:
            p = clmul_int(p, s_symbolic(i))
        i += 1
    return p


@pytest.mark.parametrize("m", range(0, 9))
def test_basis_cvt_is_the_definition(m):
    # for each monomial x^j: sum_k g_k X_k(x) == x^j (1-bit coefficients; the map is GF(2)-linear
    # and acts identically on every bit of a word, "rely on the simple form of s_i" P:516-517)
    n = 1 << m
    X = [X_poly(k) for k in range(n)]
    assert all(X[k].bit_length() - 1 == k for k in range(n))    # deg X_k = k
    for j in range(n):
        f = np.zeros(n, dtype=np.uint64)
        f[j] = 1
        g = O.basis_cvt(f)
        acc = 0
        for k in range(n):
            if g[k]:
                acc ^= X[k]
        assert acc == 1 << j


def test_spec_and_appendix_b_examples():
    import json
    import os
    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    # S:349 (tests/golden/spec_examples.json): x^2 -> X_2 + X_1
    ex = json.load(open(os.path.join(gdir, "spec_examples.json")))["basis_cvt"]
    assert list(O.basis_cvt(np.array(ex["in"], dtype=np.uint64))) == ex["out"]
    # App. B (tests/golden/appendix_b_schedule.json): n = 16 -> 4 layers with equal XOR counts:
    # divide by x^8+x^2 (d=6), then x^4+x on both halves (d=3), then y^2+y "4 positions apart", then x^2+x
    # on 4 chunks.
    g = json.load(open(os.path.join(gdir, "appendix_b_schedule.json")))
    tr = O.cvt_trace(g["m"])
    assert tr == [tuple(x) for x in g["steps"]]
    layers = [8, 4 + 4, 8, 2 * 4]
    assert len(set(layers)) == 1


@pytest.mark.parametrize("m,w", [(1, 1), (5, 1), (10, 1), (13, 2), (7, 2)])
def test_basis_cvt_roundtrip_and_linearity(m, w):
    f = splitmix64(31 + m, (1 << m) * w)
    g = O.basis_cvt(f, w)
    assert np.array_equal(O.ibasis_cvt(g, w), f)
    f2 = splitmix64(77 + m, (1 << m) * w)
    assert np.array_equal(O.basis_cvt(f ^ f2, w), g ^ O.basis_cvt(f2, w))


def test_basis_cvt_zero_extension_commutes():
    # converting 2^p words then zero-extending == converting the zero-padded 2^m vector
    for p, m in [(3, 5), (6, 9), (10, 11)]:
        f = splitmix64(3, 1 << p)
        small = O.basis_cvt(f)
        big = np.zeros(1 << m, dtype=np.uint64)
        big[: 1 << p] = f
        want = np.zeros(1 << m, dtype=np.uint64)
        want[: 1 << p] = small
        assert np.array_equal(O.basis_cvt(big), want)


def horner(coeffs, alpha):
    acc = 0
    for c in reversed(coeffs):
        acc = O.tower_mul(acc, alpha) ^ c
    return acc


@pytest.mark.parametrize("m", [1, 2, 3, 5, 6])
def test_fft_evaluates_at_tower_points(m):
    # FFT(BasisCvt(f))[i] = f(phi_v(i)) (Alg. 1 output, natural order, R2)
    n = 1 << m
    coeffs = [R.getrandbits(128) for _ in range(n)]
    f = np.array([[c & (2**64 - 1), c >> 64] for c in coeffs], dtype=np.uint64)
    g = O.basis_cvt(f.reshape(-1), 2).reshape(-1, 2)
    e = O.fft(g)
    for i in range(n):
        assert int(e[i, 0]) | (int(e[i, 1]) << 64) == horner(coeffs, i)


def test_fft_special_cases():
    # size 2: (g0, g1) -> (g0, g0 ^ g1); constant input -> constant output
    g = np.array([[5, 1], [9, 2]], dtype=np.uint64)
    assert np.array_equal(O.fft(g), np.array([[5, 1], [5 ^ 9, 3]], dtype=np.uint64))
    m = 7
    g = np.zeros((1 << m, 2), dtype=np.uint64)
    g[0] = [123, 456]
    assert np.all(O.fft(g) == g[0])
    # FFT(e_k)[i] = X_k(phi_v(i)) = 0 iff i < 2^msb(k) (s_j vanishes exactly on V_j)
    for k in [1, 2, 3, 5, 17, 64, 100]:
        g = np.zeros((1 << m, 2), dtype=np.uint64)
        g[k, 0] = 1
        e = O.fft(g)
        zero = ~np.any(e != 0, axis=1)
        msb = k.bit_length() - 1
        assert np.array_equal(zero, np.arange(1 << m) < (1 << msb))


@pytest.mark.parametrize("m", [1, 4, 9, 12])
def test_fft_roundtrip_and_linearity(m):
    g = splitmix64(40 + m, 2 << m).reshape(-1, 2)
    e = O.fft(g)
    assert np.array_equal(O.ifft(e), g)
    g2 = splitmix64(90 + m, 2 << m).reshape(-1, 2)
    assert np.array_equal(O.fft(g ^ g2), e ^ O.fft(g2))


# ---------------------------------------------------------------- Alg. 5 end to end
@pytest.mark.parametrize("bits", [1, 2, 63, 64, 65, 127, 128, 129, 200, 511, 512, 513])
def test_alg5_vs_brute_small(bits):
    a, b = operand_pair(bits, seed=bits)
    assert np.array_equal(O.alg5_mul(a, bits, b, bits), brute_mul_words(a, b))


def test_alg5_unequal_and_ragged():
    for ab, bb in [(1, 1000), (64 * 7 + 3, 64 * 2), (5000, 130), (64, 64 * 64 + 1), (3, 2)]:
        a, b = operand(ab, seed=ab), operand(bb, seed=bb + 1)
        c = O.alg5_mul(a, ab, b, bb)
        assert np.array_equal(c, brute_mul_words(a, b))
        assert np.array_equal(O.alg5_mul(b, bb, a, ab), c)       # commutativity


def test_alg5_ignores_bits_above_length():
    a, b = operand_pair(100)
    a_dirty = a.copy()
    a_dirty[-1] |= np.uint64(0xFFFF << 40)
    assert np.array_equal(O.alg5_mul(a_dirty, 100, b, 100), O.alg5_mul(a, 100, b, 100))


def test_alg5_zero_length_and_identity():
    a = operand(300)
    z = O.alg5_mul(a, 300, np.zeros(1, np.uint64), 0)
    assert len(z) == 5 and not z.any()
    one = np.array([1], dtype=np.uint64)
    assert np.array_equal(O.alg5_mul(a, 300, one, 1)[: len(a)], a)   # a * 1 = a
    zero = np.array([0], dtype=np.uint64)
    assert not O.alg5_mul(a, 300, zero, 1).any()                      # a * 0 = 0


def test_alg5_closed_forms():
    bits = 1 << 14
    a = operand(bits, seed=9)
    assert np.array_equal(O.alg5_mul(a, bits, a, bits), square_closed_form(a))   # Frobenius
    for k in [0, 1, 63, 64, 1000, bits - 1]:
        xk = np.zeros(bits // 64, dtype=np.uint64)
        xk[k // 64] = np.uint64(1 << (k % 64))
        assert np.array_equal(O.alg5_mul(a, bits, xk, bits), shift_closed_form(a, k, 2 * (bits // 64)))
        xk[0] ^= np.uint64(1)           # a * (x^k + 1) = a ^ (a << k)   (k > 0)
        if k:
            want = shift_closed_form(a, k, 2 * (bits // 64))
            want[: len(a)] ^= a
            assert np.array_equal(O.alg5_mul(a, bits, xk, bits), want)


def test_alg5_c1_vs_brute():
    bits = 1 << 16
    a, b = operand_pair(bits)
    assert np.array_equal(O.alg5_mul(a, bits, b, bits), brute_mul_words(a, b))


def test_alg5_stage_invariants():
    bits = 1 << 12
    a, b = operand_pair(bits, seed=3)
    c, st = O.alg5_mul(a, bits, b, bits, stages=True)
    N = len(st["prod"])
    # upper half of the novel-basis spectra is zero (operands have N/2 blocks) -> FFT fan-out
    assert not st["cvt_a"][N // 2:].any() and not st["cvt_b"][N // 2:].any()
    assert np.array_equal(O.fft(st["cvt_a"]), st["fft_a"])
    assert np.array_equal(O.ifft(st["prod"]), st["ifft"])
    # every pointwise product equals the tower product of the two spectra
    for i in [0, 1, 7, N - 1]:
        x = int(st["fft_a"][i, 0]) | int(st["fft_a"][i, 1]) << 64
        y = int(st["fft_b"][i, 0]) | int(st["fft_b"][i, 1]) << 64
        p = int(st["prod"][i, 0]) | int(st["prod"][i, 1]) << 64
        assert O.tower_mul(x, y) == p


def test_alg5_mod_p_medium():
    bits = 1 << 18
    a, b = operand_pair(bits, seed=12)
    c = O.alg5_mul(a, bits, b, bits)
    assert O.check_mod_p(a, b, c, O.random_irreducibles(4, seed=1))
    assert np.array_equal(c, O.mul_karatsuba(a, b))
