"""O1 brute force and O5 closed forms in pure Python integers -- TEST INFRASTRUCTURE ONLY.

A polynomial over GF(2) is a Python int whose bit i is the coefficient of x^i (§2.1,
P:211-214: "represented in bit sequence").  The product is the definition
c_k = XOR_{i+j=k} a_i b_j: for every set bit i of a, add b * x^i.
"""
from __future__ import annotations

import numpy as np


def words_to_int(w) -> int:
    w = np.asarray(w, dtype=np.uint64)
    return int.from_bytes(w.astype("<u8").tobytes(), "little")


def int_to_words(x: int, n: int) -> np.ndarray:
    return np.frombuffer(x.to_bytes(8 * n, "little"), dtype="<u8").astype(np.uint64)


def clmul_int(a: int, b: int) -> int:
    """Carry-less product by the definition (shift-and-xor over the set bits of the smaller one)."""
    if a.bit_count() > b.bit_count():
        a, b = b, a
    r = 0
    while a:
        low = a & -a
        r ^= b << (low.bit_length() - 1)
        a ^= low
    return r


def brute_mul_bits(a_bits_list, b_bits_list):
    """Bit-level O(d^2) definition on coefficient lists (root of trust for tiny sizes)."""
    c = [0] * (len(a_bits_list) + len(b_bits_list))
    for i, ai in enumerate(a_bits_list):
        for j, bj in enumerate(b_bits_list):
            c[i + j] ^= ai & bj
    return c


def brute_mul_words(a, b) -> np.ndarray:
    """Product of word arrays via Python-int shift-and-xor; returns len(a)+len(b) words."""
    return int_to_words(clmul_int(words_to_int(a), words_to_int(b)), len(a) + len(b))


# ---------------------------------------------------------------- O5 closed forms (exact, O(n))
def square_closed_form(a) -> np.ndarray:
    """a^2 over GF(2): c_{2i} = a_i, odd coefficients zero (Frobenius); 2n words."""
    a = np.asarray(a, dtype=np.uint64)
    out = np.zeros(2 * len(a), dtype=np.uint64)
    # spread each 32-bit half of a word into 64 bits (bit i -> bit 2i)
    for half in range(2):
        x = (a >> np.uint64(32 * half)) & np.uint64(0xFFFFFFFF)
        y = np.zeros_like(x)
        for i in range(32):
            y |= ((x >> np.uint64(i)) & np.uint64(1)) << np.uint64(2 * i)
        out[half::2] = y
    return out


def shift_closed_form(a, k: int, nout: int) -> np.ndarray:
    """a * x^k as nout words."""
    return int_to_words(words_to_int(a) << k, nout)
