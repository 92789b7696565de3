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
    assert G.gf2x_plan((1 << 28) + 64, 1 << 10)["trunc_j"] == 12    # a = H + 1 words, b short
    assert G.gf2x_plan((1 << 28) - 64 * 16, 1 << 10)["trunc_j"] == -1   # L = 2^22 - 1: L - H = 2^21 - 1, too far above H
    assert G.gf2x_plan((1 << 29) + 64, 64)["trunc_j"] == 12        # an operand reaching past H by a short tail
    assert G.gf2x_plan((1 << 28) + 64 * 5000, 64)["trunc_j"] == 13


def test_plan_rejects_empty():
    with pytest.raises(G.Gf2xError):
        G.gf2x_plan(0, 64)


def lucas_terms(p):
    return [q for q in range(p) if (q & p) == q]


@pytest.mark.parametrize("ab,bb", SIZES + [(((1 << 16) + 5) * 64, 3 * 64), (((1 << 16) + (1 << 14)) * 64, 64),
                                           (((1 << 16) + (1 << 14) + 1) * 64, 64), ((1 << 22) + 64, (1 << 22) + 64)])
def test_split_conversion_plan(ab, bb):
    # DESIGN.md R22: one product, a conversion length n in (2^p, 2^p + 2^j] with j <= p - 2 and 2^(p+1) >= 2^16
    # units is split into a 2^p and a 2^j conversion
    p = G.gf2x_plan(ab, bb)
    na, nb = (ab + 63) // 64, (bb + 63) // 64

    def want(n, mfull):
        if mfull < 16 or n <= 1 << (mfull - 1):
            return None
        j = max(0, (n - (1 << (mfull - 1)) - 1).bit_length())
        return [mfull - 1, j] if j <= mfull - 3 else None

    assert p["split"]["a"] == want(na, p["ma"])
    assert p["split"]["b"] == want(nb, p["mb"])
    assert p["split"]["icvt"] == want(na + nb - 1, p["m"])


def test_split_fold_targets_stay_in_the_lower_half():
    # the s_p shift terms x^(2^q), q a proper subset of p, move a tail of 2^j (j <= p - 2) to [2^q, 2^q + 2^j),
    # below 2^p for every p (so the two conversions stay independent)
    for p in range(15, 33):
        for q in lucas_terms(p):
            assert (1 << q) + (1 << (p - 2)) <= 1 << p


@pytest.mark.parametrize("bits", [(1 << 23) + 192, (1 << 24) + 64, (1 << 28) + 64, (1 << 28) + (1 << 23)])
def test_truncated_launch_count_is_consistent(bits):
    # the truncated path launches fewer kernels' worth of work than the full transform but at least its lower
    # half's passes; the count is what bench.py reports as gpu_launches (checked against the profiler on the GPU)
    n = G.gf2x_launch_count(bits, bits)
    p = G.gf2x_plan(bits, bits)
    assert p["trunc_j"] >= 12
    assert 20 <= n <= 60
