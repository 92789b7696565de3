"""Host check of the split conversion schedule of k_small (csrc/small.cuh sm_conv_op / sm_low_block, gf2x.cu
seg_cvt): BasisCvt's op list for 2^mm units is [top run][low block: levels <= K][high block: bits >= K], and
the kernel runs the low block AFTER the high block, window (2^K units) by window and on each 2^mloc-unit point
segment separately (the two blocks commute: Kronecker factors); the inverse runs the inverted low block on its
segment BEFORE the rest.  The schedule is
executed here with plain sweeps (the kernel's sm_sweep, restated) over the planner's op list (cvt_ops,
restated) and compared with the oracle's Alg. 3 BasisCvt / iBasisCvt on random data, segment by segment
(so a wrong op list, sweep or reordering fails against the oracle, not against itself)."""
import numpy as np
import pytest

import oracle as O
from gf2x_synth import splitmix64


def cvt_ops(m, sigma=0, out=None):
    out = [] if out is None else out
    if m <= 1:
        return out
    K = 1
    while 2 * K <= m - 1:
        K *= 2
    for lev in range(m, K, -1):
        out.append((lev + sigma, K))
    cvt_ops(K, sigma, out)
    cvt_ops(m - K, sigma + K, out)
    return out


def sweep(s, off, mm, lg, K, A):
    h = 1 << (lg - 1)
    u = h >> K
    d = h - u
    for seg in range(1 << (mm - lg)):
        b = off + (seg << lg)
        if A:
            s[b + h: b + h + u] ^= s[b + h + d: b + h + d + u]
        else:
            s[b + u: b + h] ^= s[b + u + d: b + h + d]


def split_info(mm, m, QB):
    """(split, ntop, nlow, K) as gf2x.cu's seg_cvt."""
    K = 1
    while 2 * K <= mm - 1:
        K *= 2
    if mm <= 2 or K > m - QB:
        return 0, 0, 0, 0
    return 1, mm - K, len(cvt_ops(K)), K


@pytest.mark.parametrize("m,QB", [(11, 2), (10, 2), (11, 1), (9, 1), (8, 1), (9, 2), (7, 1), (11, 0), (9, 0), (6, 0)])
@pytest.mark.parametrize("mm_off", [0, 1, 2])
def test_forward_segments_match_oracle(m, QB, mm_off):
    """Every CTA q: CTA-wide steps (top run, then high block; all ops if not split) on the whole operand unless
    its segment lies past it, then the low block window by window on its segment's part of the operand."""
    mm = m - mm_off   # operand of 2^mm words zero-extended to 2^m
    N, mloc = 1 << m, m - QB
    f = np.zeros(N, np.uint64)
    f[: 1 << mm] = splitmix64(1000 * m + mm, 1 << mm)
    want = np.zeros(N, np.uint64)
    want[: 1 << mm] = O.basis_cvt(f[: 1 << mm])
    ops = cvt_ops(mm)
    split, ntop, nlow, K = split_info(mm, m, QB)
    cta_ops = list(range(ntop)) + list(range(ntop + nlow, len(ops))) if split else list(range(len(ops)))
    for q in range(1 << QB):
        s = f.copy()
        sbase = q << mloc
        if sbase < (1 << mm):
            for oi in cta_ops:
                lg, Kop = ops[oi]
                for A in (True, False):
                    sweep(s, 0, mm, lg, Kop, A)
            if split:
                lo = sbase
                hi = min(lo + (1 << mloc), 1 << mm)
                for w in range(lo, hi, 1 << K):
                    for oi in range(ntop, ntop + nlow):
                        lg, Kop = ops[oi]
                        for A in (True, False):
                            sweep(s, w, K, lg, Kop, A)
        assert np.array_equal(s[sbase: sbase + (1 << mloc)], want[sbase: sbase + (1 << mloc)]), (q, split)


@pytest.mark.parametrize("m,QB", [(11, 2), (10, 2), (11, 1), (9, 1), (8, 1), (9, 2), (11, 0), (7, 0)])
def test_inverse_segments_match_oracle(m, QB):
    N, mloc = 1 << m, m - QB
    g = splitmix64(77 + m, N)
    want = O.ibasis_cvt(g)
    ops = cvt_ops(m)
    mode, ntop, nlow, K = split_info(m, m, QB)
    # every CTA inverts the low block window by window on its own segment, then the array is gathered
    s = g.copy()
    if mode == 1:
        for q in range(1 << QB):
            for w in range(q << mloc, (q + 1) << mloc, 1 << K):
                for oi in range(ntop + nlow - 1, ntop - 1, -1):
                    lg, Kop = ops[oi]
                    for A in (False, True):
                        sweep(s, w, K, lg, Kop, A)
        nhigh = len(ops) - ntop - nlow
        rest = [len(ops) - 1 - i for i in range(nhigh)] + [ntop - 1 - i for i in range(ntop)]
    else:
        rest = list(range(len(ops) - 1, -1, -1))
    for oi in rest:
        lg, Kop = ops[oi]
        for A in (False, True):
            sweep(s, 0, m, lg, Kop, A)
    assert np.array_equal(s, want), mode

