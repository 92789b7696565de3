"""Host-side planner (gf2x_plan, no GPU): the passes the CUDA path enqueues cover exactly the paper's work.

  * BasisCvt / iBasisCvt passes: their Taylor steps, concatenated in execution order, are Alg. 3's steps
    (largest-K split, R4-R6) -- with each node's inner conversions (index window inside
    [sigma, sigma+K)) before its outer one ([sigma+K, sigma+m)), the commutation of DESIGN.md R14 -- and as a
    multiset exactly the steps of the paper's order;
  * FFT_LCH: the table passes and the bit-sliced bottom cover layers [0, m) once, top-down, each pass's
    column bits below its layers, at most 6 layers in the changeRepr pass and 7 below.
"""
import random

import pytest

import paper_1708_09746_b200 as G


def K_of(m):
    K = 1
    while 2 * K <= m - 1:
        K *= 2
    return K


def steps_paper(m, sigma=0):
    """Alg. 3 in the paper's order: Taylor levels, outer BasisCvt(h(y)), then the inner BasisCvt(q_i)."""
    if m <= 1:
        return []
    K = K_of(m)
    out = [(l + sigma, K) for l in range(m, K, -1)]
    out += steps_paper(m - K, sigma + K)
    out += steps_paper(K, sigma)
    return out


def steps_inner_first(m, sigma=0):
    if m <= 1:
        return []
    K = K_of(m)
    return [(l + sigma, K) for l in range(m, K, -1)] + steps_inner_first(K, sigma) + steps_inner_first(m - K, sigma + K)


def flatten(passes):
    return [tuple(op) for p in passes for op in p["ops"]]


SIZES = [(1, 1), (64, 64), (65, 64), (3000, 17), (1 << 14, 1 << 14), (1 << 16, 1 << 16), (1 << 20, 1000),
         (1 << 24, 1 << 24), (1 << 28, 1 << 28), (1 << 29, 1 << 29), ((1 << 28) + 64, 1 << 20), (1 << 32, 1 << 32)]


@pytest.fixture(scope="module", autouse=True)
def _lib():
    G.load()


@pytest.mark.parametrize("ab,bb", SIZES + [(random.Random(i).randrange(1, 1 << 30), random.Random(i + 99).randrange(1, 1 << 30))
                                           for i in range(8)])
def test_plan_covers_the_method(ab, bb):
    p = G.gf2x_plan(ab, bb)
    na, nb = (ab + 63) // 64, (bb + 63) // 64
    m = max(0, (na + nb - 2).bit_length())
    assert p["m"] == m and p["N"] == 1 << m
    # conversions: Alg. 3 steps, inner-first order, and the same multiset as the paper's order
    for key, mm in (("cvt_a", p["ma"]), ("cvt_b", p["mb"]), ("icvt", m)):
        got = flatten(p[key])
        assert got == steps_inner_first(mm), key
        assert sorted(got) == sorted(steps_paper(mm)), key
        for ps in p[key]:
            if ps["kind"] == "res":   # one K per residue run, consecutive descending levels
                assert len({k for _, k in ps["ops"]}) == 1
                assert [l for l, _ in ps["ops"]] == list(range(ps["ops"][0][0], ps["ops"][0][0] - len(ps["ops"]), -1))
    # FFT: table passes then the bottom cover [0, m) exactly once, top-down
    top = m
    for i, (c, k_lo, k_hi) in enumerate(p["fft"]):
        assert k_hi == top and k_lo < k_hi and c <= k_lo
        assert k_hi - k_lo <= (6 if i == 0 else 7)
        top = k_lo
    assert top == p["bottom"] == min(m, 6 if m > 10 else 5)


def test_truncation_eligibility():
    # L just above a power of two, both operands in the lower half: truncated with the smallest 2^j >= L - H
    p = G.gf2x_plan((1 << 28) + 64, (1 << 28) + 64)
    assert p["m"] == 24 and p["trunc_j"] == 12
    p = G.gf2x_plan((1 << 28) + (1 << 23), (1 << 28) + (1 << 23))
    assert p["trunc_j"] == 18   # L - H = 2^18 - 1
    assert G.gf2x_plan(1 << 29, 1 << 29)["trunc_j"] == -1          # exact power of two
    assert G.gf2x_plan((1 << 28) + 64, 1 << 10)["trunc_j"] == -1   # L <= H
    assert G.gf2x_plan((1 << 29) + 64, 64)["trunc_j"] == -1        # an operand beyond the lower half


def test_plan_rejects_empty():
    with pytest.raises(G.Gf2xError):
        G.gf2x_plan(0, 64)
