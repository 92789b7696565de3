"""Pins for oracle O1/O2 (carry-less multiplication) -- PAPER.md §2.1 P:211-214 definition
c_k = XOR_{i+j=k} a_i b_j, and SPEC.md worked examples."""
import random

import numpy as np
import pytest

import oracle as O
from oracle.brute import brute_mul_bits, brute_mul_words, clmul_int, words_to_int, int_to_words
from gf2x_synth import operand_pair, splitmix64


def test_spec_examples():
    # S:106 clmul 0x3 * 0x3 = 0x5 ; S:42-44 (x+1)^2 = x^2+1, 0b111 * 0b11 = 0b1001 (tests/golden/spec_examples.json)
    import json
    import os
    ex = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "spec_examples.json")))
    for a, b, r in ex["clmul"]:
        assert O.clmul64(a, b) == r
        assert O.clmul64(a, b, portable=True) == r
        assert clmul_int(a, b) == r
    assert brute_mul_bits([1, 1, 1], [1, 1]) == [1, 0, 0, 1, 0]


def test_clmul64_hw_vs_portable_vs_python():
    rng = random.Random(1)
    for _ in range(2000):
        a, b = rng.getrandbits(64), rng.getrandbits(64)
        want = clmul_int(a, b)
        assert O.clmul64(a, b) == want
        assert O.clmul64(a, b, portable=True) == want
    assert O.clmul64(2**64 - 1, 2**64 - 1) == clmul_int(2**64 - 1, 2**64 - 1)


def test_int_brute_vs_bit_brute():
    rng = random.Random(2)
    for _ in range(50):
        la, lb = rng.randint(1, 70), rng.randint(1, 70)
        a = [rng.randint(0, 1) for _ in range(la)]
        b = [rng.randint(0, 1) for _ in range(lb)]
        ai = sum(x << i for i, x in enumerate(a))
        bi = sum(x << i for i, x in enumerate(b))
        c = brute_mul_bits(a, b)
        assert sum(x << i for i, x in enumerate(c)) == clmul_int(ai, bi)


@pytest.mark.parametrize("na,nb", [(1, 1), (1, 7), (3, 5), (16, 16), (33, 33), (40, 17)])
def test_schoolbook_vs_brute(na, nb):
    a = splitmix64(11, na)
    b = splitmix64(12, nb)
    assert np.array_equal(O.mul_schoolbook(a, b), brute_mul_words(a, b))


@pytest.mark.parametrize("n", [1, 31, 32, 33, 65, 100, 257, 1024])
def test_karatsuba_vs_schoolbook(n):
    a = splitmix64(21, n)
    b = splitmix64(22, n)
    assert np.array_equal(O.mul_karatsuba(a, b), O.mul_schoolbook(a, b))


def test_mul_word_vs_full_product():
    a, b = operand_pair(64 * 300 + 17)
    full = O.mul_schoolbook(a, b)
    for w in [0, 1, 2, 150, 299, 300, 301, 598, 599, len(full) - 1]:
        assert O.mul_word(a, b, w) == int(full[w])


def test_karatsuba_vs_python_int():
    # 2^17-bit operands: Karatsuba oracle vs Python big-int shift-xor (independent code paths)
    a, b = operand_pair(1 << 17)
    want = brute_mul_words(a, b)
    assert np.array_equal(O.mul_karatsuba(a, b), want)


def test_mod_p_detects_errors():
    primes = O.random_irreducibles(4, seed=99)
    for r in primes:
        assert O.is_irreducible64(r)
    # x^64 + x^4 + x^3 + x + 1 is irreducible (standard GF(2^64) modulus); x^64 + x^2 + 1 = (x^32+x+1)^2
    assert O.is_irreducible64(0b11011)
    assert not O.is_irreducible64(0b101)
    a, b = operand_pair(1 << 14)
    c = O.mul_schoolbook(a, b)
    assert O.check_mod_p(a, b, c, primes)
    for w, bit in [(0, 0), (100, 63), (len(c) - 2, 5)]:
        bad = c.copy()
        bad[w] ^= np.uint64(1 << bit)
        assert not O.check_mod_p(a, b, bad, primes)
