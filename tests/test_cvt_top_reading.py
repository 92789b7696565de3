"""Host-side check of the algebra k_cvt_top relies on (cvt.cuh): the top Taylor run of Alg. 3 (Alg. 2's
divisions "by repeatedly subtracting", levels q .. K+1, R4) equals, on residue classes
i = r M + c (M = 2^K - 1), the superset-sum transform over the row bits for the generic classes
c >= 2^B - 1 + 2^(B-1) (B = q - K) and the phase-A / phase-B sweeps for the others -- in both directions.
Small analogues (K = 4, 8) of the kernel's K = 16 case, against the plain sequential loop."""
import random

import pytest

def taylor_seq(f, q, K, inverse=False):
    f = f[:]
    levels = list(range(q, K, -1))
    if inverse: levels = levels[::-1]
    for lg in levels:
        h = 1 << (lg - 1); u = h >> K; d = h - u
        for s in range(0, len(f), 1 << lg):
            rng = range(2*h - 1, h - 1, -1) if not inverse else range(h, 2*h)
            for i in rng:
                f[s + i - d] ^= f[s + i]
    return f

def top_kernel(f, q, K, inverse=False):
    f = f[:]
    M = (1 << K) - 1; B = q - K; span = 1 << q
    cgen = (1 << B) - 1 + (1 << (B - 1))
    for c in range(M):
        rows = [r for r in range((span - 1 - c) // M + 1)]
        col = [f[r*M + c] for r in rows]
        if c >= cgen:
            assert len(col) == 1 << B, (c, len(col))
            for b in range(B):
                for r in range(len(col)):
                    if not (r >> b) & 1: col[r] ^= col[r | (1 << b)]
        else:
            nl = q - K
            for o in range(nl):
                lg = K + 1 + o if inverse else q - o
                u = 1 << (lg - 1 - K); h = 1 << (lg - 1); segm = (1 << lg) - 1
                for ph in range(2):
                    A = (ph == 0) != inverse
                    lo, ln = (h, u) if A else (u, h - u)
                    new = col[:]
                    for r in rows:
                        i = r*M + c
                        if ((i & segm) - lo) % (1 << 32) < ln:
                            new[r] = col[r] ^ col[r + u]
                    col = new
        for r in rows: f[r*M + c] = col[r]
    return f


@pytest.mark.parametrize("q,K", [(7, 4), (8, 4), (9, 4), (6, 4), (10, 8), (11, 8)])
@pytest.mark.parametrize("inverse", [False, True])
def test_top_run_reading(q, K, inverse):
    random.seed(q * 100 + K)
    f = [random.getrandbits(16) for _ in range(1 << q)]
    assert taylor_seq(f, q, K, inverse) == top_kernel(f, q, K, inverse)
    assert taylor_seq(taylor_seq(f, q, K, False), q, K, True) == f
