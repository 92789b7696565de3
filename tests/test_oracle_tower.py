"""Pins for oracle O3 field arithmetic: the tower TGF(2^(2^l)) (§3.2), the
vanishing polynomials s_k (Def. 2, Table 1, Prop. 1, Prop. 3
P:796-799, Fig. 2 narrative P:833-845), and changeRepr (§4.3)."""
import json
import os
import random

import pytest

import oracle as O
from oracle.brute import clmul_int

R = random.Random(7)
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def rnd(bits):
    return R.getrandbits(bits)


# ---------------------------------------------------------------- tower arithmetic
def test_spec_small_field_examples():
    # S:175-177 (tests/golden/spec_examples.json): GF(4) 0x2*0x2 = 0x3, 0x2*0x3 = 0x1 ; GF(16) 0x2*0x8 = 0xc
    for e in golden("spec_examples.json")["tower"]:
        assert O.tower_mul(e["a"], e["b"], e["level"]) == e["r"]
        assert O.tower_mul(e["a"], e["b"], e["level"], bits_only=True) == e["r"]


def test_notation_example():
    # P:668-686 (tests/golden/tower_notation.json): x_2 x_1 + x_2 + x_1 + 1 = 0xf, v_3 = x_2 x_1 = 0x8,
    # and the 16 elements 0x00..0x0f of GF(256) are closed under the product (the subfield GF(16))
    g = golden("tower_notation.json")
    x1, x2 = g["generators"]["x1"], g["generators"]["x2"]
    x2x1 = O.tower_mul(x2, x1, 2)
    assert x2x1 == g["v"][3]
    assert x2x1 ^ x2 ^ x1 ^ 1 == g["x2x1_plus_x2_plus_x1_plus_1"]
    n = g["subfield_of_gf256"]
    assert all(O.tower_mul(a, b, 3) < n for a in range(n) for b in range(n))


@pytest.mark.parametrize("k", range(1, 8))
def test_defining_relations(k):
    # x_k^2 + x_k = x_1 ... x_(k-1)  (= 1 for k = 1).  x_k = v_(2^(k-1)) = 1 << 2^(k-1);
    # x_1 ... x_(k-1) = v_(2^(k-1)-1) = 1 << (2^(k-1) - 1).
    xk = 1 << (1 << (k - 1))
    prod = 1 << ((1 << (k - 1)) - 1)
    for bits_only in (False, True):
        assert O.tower_mul(xk, xk, 7, bits_only) ^ xk == prod


def test_table_vs_bit_recursion():
    # the GF(256)-bottomed product equals the pure AND/XOR recursion at every level
    for level in range(1, 8):
        for _ in range(40 if level < 7 else 15):
            a, b = rnd(1 << level), rnd(1 << level)
            assert O.tower_mul(a, b, level) == O.tower_mul(a, b, level, bits_only=True)


def test_field_axioms_sampled():
    for _ in range(100):
        a, b, c = rnd(128), rnd(128), rnd(128)
        ab = O.tower_mul(a, b)
        assert ab == O.tower_mul(b, a)
        assert O.tower_mul(ab, c) == O.tower_mul(a, O.tower_mul(b, c))
        assert O.tower_mul(a, b ^ c) == ab ^ O.tower_mul(a, c)
        assert O.tower_mul(a, 1) == a


def test_gf256_all_invertible():
    for a in range(1, 256):
        assert any(O.tower_mul(a, b, 3) == 1 for b in range(1, 256))


def test_subfield_embedding():
    # "the representation of each field is embedded in the lower bit(s)"
    for _ in range(200):
        a, b = rnd(4), rnd(4)
        assert O.tower_mul(a, b, 7) == O.tower_mul(a, b, 2) < 16
        a, b = rnd(16), rnd(16)
        assert O.tower_mul(a, b, 7) == O.tower_mul(a, b, 4) < 1 << 16


@pytest.mark.parametrize("sub", [2, 3, 4, 5])
def test_prop2_limbwise(sub):
    # Prop. 2: a in TGF(2^128) times b in TGF(2^(2^sub)) is 128/2^sub independent
    # products of the 2^sub-bit limbs.
    w = 1 << sub
    for _ in range(30):
        a, b = rnd(128), rnd(w)
        limbs = 0
        for i in range(128 // w):
            limbs |= O.tower_mul((a >> (w * i)) & ((1 << w) - 1), b, sub) << (w * i)
        assert O.tower_mul(a, b) == limbs


def test_prop3():
    # Prop. 3: v_i^2 + v_i in V_i, i.e. < 2^i
    for i in range(128):
        v = 1 << i
        assert O.tower_mul(v, v) ^ v < (1 << i) if i else O.tower_mul(v, v) ^ v == 0


# ---------------------------------------------------------------- s_k
def s_exponents(i):
    """s_i as the set {j : x^(2^j) is a term}, from s_0 = x and s_(k+1) = s_k^2 + s_k
    (recursivity P:327); squaring maps x^(2^j) to x^(2^(j+1)) in characteristic 2."""
    s = {0}
    for _ in range(i):
        s = {j + 1 for j in s} ^ s
    return s


def s_symbolic(i):
    """s_i as a GF(2)[x] polynomial (Python int, bit e = x^e)."""
    return sum(1 << (1 << j) for j in s_exponents(i))


def test_table1():
    # Table 1, exponent sets typed from the paper (tests/golden/table1_s_i.json)
    table1 = golden("table1_s_i.json")["s_i_exponents"]
    assert len(table1) == 8
    for i, exps in table1.items():
        assert s_symbolic(int(i)) == sum(1 << e for e in exps)
    # "minimal two terms iff i is a power of 2"
    for i in range(1, 200):
        assert (len(s_exponents(i)) == 2) == (i & (i - 1) == 0)


def _eval_linearized(poly, alpha):
    """sum over exponents 2^j of alpha^(2^j), by repeated tower squaring."""
    acc, j, sq = 0, 0, alpha
    while (1 << j) < poly.bit_length():
        if (poly >> (1 << j)) & 1:
            acc ^= sq
        sq = O.tower_mul(sq, sq)
        j += 1
    return acc


def test_s_eval_matches_table1_polynomials():
    # the oracle's k-fold s_1 equals evaluating the Table-1 polynomial at random tower points
    for i in range(0, 9):
        poly = s_symbolic(i)
        for _ in range(8):
            a = rnd(128)
            assert O.s_eval(i, a) == _eval_linearized(poly, a)


def test_s_vanishes_on_V_i():
    # Def. 2 + Claim 1: s_i vanishes exactly on V_i = span(v_0..v_(i-1)) = [0, 2^i)
    for i in range(0, 9):
        for a in range(1 << i):
            assert O.s_eval(i, a) == 0
        for a in [1 << i, (1 << i) | 3, (1 << (i + 1)) - 1]:
            assert O.s_eval(i, a) != 0


def test_prop1_s_k_of_v_k_is_one():
    # Prop. 1: s_k(v_k) = 1
    for k in range(0, 100):
        assert O.s_eval(k, 1 << k) == 1


def test_multiplier_shortening():
    # s_k(alpha) is k bits shorter than alpha and independent of its low k bits
    for _ in range(50):
        k = R.randint(0, 31)
        a = rnd(32)
        if a >> k == 0:
            continue
        r = O.s_eval(k, a)
        assert r.bit_length() == a.bit_length() - k
        assert O.s_eval(k, a ^ rnd(k) if k else a) == r


def test_fig2_multipliers():
    # Fig. 2 narrative: 16 points, degree-7 input.  Layer s_2 at alpha in {0, 0x8}:
    # {0, 0x2}; layer s_1 at {0, 0x4, 0x8, 0xc}: {0, 0x2, 0x5, 0x7}; layer s_0: {0, 0x2, ..., 0xe}.
    g = golden("fig2_multipliers.json")
    m = g["m"]
    for k, want in g["layer_multipliers"].items():   # top layer [0]: alpha = 0 -> fan-out
        assert [O.fft_constant(m, int(k), j) for j in range(len(want))] == want, k
    assert O.s_eval(1, 0x8) == g["s1_of_0x8"]


def test_multiply_count_bound():
    # "at each of log n layers there are n/2 butterflies for a total of 1/2 n log n multiplications"
    # (P:619-620): the nontrivial multiplier count never exceeds it.
    for m in range(1, 14):
        assert O.fft_mult_count(m) <= (1 << (m - 1)) * m


# ---------------------------------------------------------------- GF(2^128) and changeRepr
G = (1 << 128) | 0x87  # z^128 + z^7 + z^2 + z + 1


def gf128_ref(a, b):
    p = clmul_int(a, b)
    for i in range(p.bit_length() - 1, 127, -1):
        if (p >> i) & 1:
            p ^= G << (i - 128)
    return p


def test_gf128_mul():
    for _ in range(100):
        a, b = rnd(128), rnd(128)
        assert O.gf128_mul(a, b) == gf128_ref(a, b)


def test_psi_generators_satisfy_defining_relations():
    # the images X_k of x_k satisfy X_1^2+X_1 = 1 and X_k^2+X_k = X_1...X_(k-1) in GF(2^128)
    prod = 1
    for k in range(1, 8):
        X = O.psi_generator(k)
        assert gf128_ref(X, X) ^ X == prod
        assert X < X ^ 1 or X == 0       # the numerically smaller root (R9)
        prod = gf128_ref(prod, X)


def test_psi_is_field_isomorphism():
    assert O.psi(1) == 1 and O.psi_inv(1) == 1
    for _ in range(60):
        u, v = rnd(128), rnd(128)
        assert O.psi(gf128_ref(u, v)) == O.tower_mul(O.psi(u), O.psi(v))
        assert O.psi_inv(O.psi(u)) == u
        assert O.psi(O.psi_inv(u)) == u


def test_psi_of_z_is_root_of_modulus():
    # psi(z) must satisfy z^128 + z^7 + z^2 + z + 1 = 0 in the tower
    t = O.psi(2)
    powers = [1]
    for _ in range(128):
        powers.append(O.tower_mul(powers[-1], t))
    assert powers[128] ^ powers[7] ^ powers[2] ^ powers[1] ^ powers[0] == 0
