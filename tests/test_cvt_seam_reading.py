"""Host-side pin of DESIGN.md R27, the closed form k_cvt_seam (cvt.cuh) computes: a complete Taylor run of
Alg. 3 (levels q .. K+1 of a 2^q-unit chunk, Alg. 2's divisions "by repeatedly subtracting") maps
each residue class c = 1 .. M (M = 2^K - 1, unit i = r M + c, rows r = 0 .. 2^B, B = q - K) to
    y[r] = XOR_{s superset of r} x[s]        (r < c)
    y[r] = XOR_{s superset of r-1} x[s+1]    (r >= c),
and the inverse run to  x_U = T y_U,  x_L = S(y on L, S(x_U on U, 0 on L) on U) on L.

The check composes the closed form with the ORACLE's own conversions of the inner and outer nodes (Alg. 3's
recursion: the run, then CVT(K) on the low K index bits and CVT(q - K) on the high bits, R14) and compares the
result with the oracle's BasisCvt / iBasisCvt of the whole chunk, so a wrong seam, a wrong shift or a wrong
inverse order fails it.  numpy only; the oracle is the reference, the closed form is written here from R27."""
import numpy as np
import pytest

import oracle as O


def _ss(a):
    """superset-sum over the bits of axis 0 (length a power of two)"""
    a = a.copy()
    n = a.shape[0]
    b = 1
    while b < n:
        v = a.reshape(n // (2 * b), 2, b, *a.shape[1:])
        v[:, 0] ^= v[:, 1]
        b *= 2
    return a


def _classes(f, q, K):
    """rows x classes matrix (rows 0 .. 2^B, classes 1 .. M) of units i = r M + c (zero beyond the chunk)"""
    M = (1 << K) - 1
    B = q - K
    r = np.arange((1 << B) + 1)[:, None]
    c = np.arange(1, M + 1)[None, :]
    i = r * M + c
    ok = i < (1 << q)
    X = np.zeros(i.shape + f.shape[1:], dtype=np.uint64)
    X[ok] = f[i[ok]]
    return X, i, ok, r, c


def seam_forward(f, q, K):
    X, i, ok, r, c = _classes(f, q, K)
    n = 1 << (q - K)
    P = _ss(X[:n])
    P[0] ^= X[n]
    Q = _ss(X[1:])
    Y = np.zeros_like(X)
    low = r < c
    sel = low[:n] if X.ndim == 2 else low[:n, :, None]
    Y[:n] = np.where(sel, P, 0)
    up = (r >= c)[1:]
    sel = up if X.ndim == 2 else up[..., None]
    Y[1:] ^= np.where(sel, Q, 0)
    g = f.copy()
    g[i[ok]] = Y[ok]
    return g


def seam_inverse(g, q, K):
    Y, i, ok, r, c = _classes(g, q, K)
    n = 1 << (q - K)
    ex = (lambda m: m) if Y.ndim == 2 else (lambda m: m[..., None])
    up = ex(r >= c)
    Qy = _ss(Y[1:])
    XU = np.zeros_like(Y)
    XU[1:] = np.where(up[1:], Qy, 0)              # x_U = T y_U (zero on L)
    V = _ss(XU[:n])                              # v = S(x_U, 0 on L): rows < 2^B
    Vn = XU[n]                                   # the extra row is only its own superset
    Wv = np.where(up[:n], V, Y[:n])              # w = (y on L, v on U)
    XL = _ss(Wv)
    XL[0] ^= Vn
    X = XU.copy()
    X[:n] = np.where(up[:n], XU[:n], XL)
    f = g.copy()
    f[i[ok]] = X[ok]
    return f


def _cvt_rest(g, q, K, inverse):
    """the inner CVT(K) (each 2^K block) and outer CVT(q-K) (stride 2^K) through the oracle"""
    w = 1 if g.ndim == 1 else g.shape[1]
    cv = O.ibasis_cvt if inverse else O.basis_cvt
    blocks = g.reshape(1 << (q - K), 1 << K, *g.shape[1:])
    inner = np.stack([cv(b.reshape(-1), w).reshape(b.shape) for b in blocks])
    cols = inner.swapaxes(0, 1)
    outer = np.stack([cv(col.reshape(-1), w).reshape(col.shape) for col in cols]).swapaxes(0, 1)
    return np.ascontiguousarray(outer).reshape(g.shape)


@pytest.mark.parametrize("q,K,w", [(13, 8, 1), (16, 8, 1), (16, 8, 2), (21, 16, 1), (15, 8, 2)])
def test_seam_closed_form_vs_oracle_cvt(q, K, w):
    rng = np.random.default_rng(q * 31 + w)
    shape = (1 << q,) if w == 1 else (1 << q, w)
    f = rng.integers(0, 1 << 63, size=shape, dtype=np.uint64)
    want = O.basis_cvt(f.reshape(-1), w).reshape(shape)
    # forward: the run first (Alg. 3 order), then the inner and outer nodes (they commute, R14)
    got = _cvt_rest(seam_forward(f, q, K), q, K, inverse=False)
    assert np.array_equal(got, want)
    # inverse: inner / outer nodes inverted first, the run last
    back = seam_inverse(_cvt_rest(want, q, K, inverse=True), q, K)
    assert np.array_equal(back, f)
    assert np.array_equal(O.ibasis_cvt(want.reshape(-1), w).reshape(shape), f)


def test_seam_is_not_plain_superset_sum():
    """the seam matters: the plain superset-sum on every class (R24's generic form) is wrong below the seam"""
    q, K = 13, 8
    f = np.random.default_rng(5).integers(0, 1 << 63, size=1 << q, dtype=np.uint64)
    X, i, ok, r, c = _classes(f, q, K)
    n = 1 << (q - K)
    P = _ss(X[:n])
    P[0] ^= X[n]
    g = f.copy()
    Y = X.copy()
    Y[:n] = P
    g[i[ok]] = Y[ok]
    want = O.basis_cvt(f, 1)
    assert not np.array_equal(_cvt_rest(g, q, K, inverse=False), want)
