"""GPU parity of App. C, the multiply through the Frobenius bijection: its bit-level BasisCvt
(gf2x_basis_cvt_bits) against the oracle's bit-level Alg. 3 (O.basis_cvt_bits, pinned in test_oracle_frob.py)
and the whole multiply (gf2x_mul_frob) against the oracle's App. C multiply, brute force and Karatsuba.
Bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from oracle.brute import brute_mul_words  # noqa: E402
from gf2x_synth import operand, operand_pair  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


@pytest.mark.parametrize("M", [6, 7, 8, 9, 11, 12, 16, 17, 20, 23])
def test_bit_basis_cvt_matches_oracle(M):
    f = operand(1 << M, seed=M + 500)
    d = dev(f)
    G.gf2x_basis_cvt_bits(d, M)
    g = host(d)
    assert np.array_equal(g, O.basis_cvt_bits(f, M))
    G.gf2x_basis_cvt_bits(d, M, inverse=True)
    assert np.array_equal(host(d), f)
    d2 = dev(g)
    G.gf2x_basis_cvt_bits(d2, M, inverse=True)
    assert np.array_equal(host(d2), O.basis_cvt_bits(g, M, inverse=True))


def test_bit_basis_cvt_sparse_and_edge_inputs():
    M = 10
    for f in [np.zeros(1 << (M - 6), np.uint64), np.full(1 << (M - 6), np.uint64(0xFFFFFFFFFFFFFFFF))]:
        d = dev(f)
        G.gf2x_basis_cvt_bits(d, M)
        assert np.array_equal(host(d), O.basis_cvt_bits(f, M))
    for t in [0, 1, 63, 64, 511, 512, 1023]:   # monomials x^t
        f = np.zeros(1 << (M - 6), np.uint64)
        f[t // 64] = np.uint64(1 << (t % 64))
        d = dev(f)
        G.gf2x_basis_cvt_bits(d, M)
        assert np.array_equal(host(d), O.basis_cvt_bits(f, M)), t
    with pytest.raises(G.Gf2xError):
        G.gf2x_basis_cvt_bits(dev(np.zeros(1, np.uint64)), 5)


def test_bit_basis_cvt_full_size_roundtrip():
    # the size the App. C multiply of two 2^29-bit operands converts (2^30 coefficients): the inverse returns
    # the input, and sampled words of a sparse input match the oracle at a size it converts in seconds
    M = 30
    f = operand(1 << M, seed=77)
    d = dev(f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.gf2x_basis_cvt_bits(d, M)
    e1.record()
    torch.cuda.synchronize()
    print(f"bit-level BasisCvt, 2^{M} coefficients: {e0.elapsed_time(e1):.2f} ms")
    G.gf2x_basis_cvt_bits(d, M, inverse=True)
    assert np.array_equal(host(d), f)


def gpu_frob(a, ab, b, bb):
    return host(G.gf2x_mul_frob(dev(a), ab, dev(b), bb))


@pytest.mark.parametrize("bits", [1, 2, 63, 64, 65, 127, 128, 129, 255, 256, 1000, 4096, 5000, 8191, 1 << 14, (1 << 14) + 3])
def test_frob_mul_square_sizes(bits):
    a, b = operand_pair(bits, seed=bits + 900)
    got = gpu_frob(a, bits, b, bits)
    assert np.array_equal(got, brute_mul_words(a, b) if bits <= 8192 else O.frob_mul(a, bits, b, bits))


@pytest.mark.parametrize("ab,bb", [(1, 1000), (1000, 1), (64, 65), (300, 4000), (128 * 16, 128 * 16 + 1), (3, 2), (5000, 130),
                                   (1 << 16, 77), (70000, 1 << 15)])
def test_frob_mul_unequal_sizes(ab, bb):
    a, b = operand(ab, seed=ab + 1), operand(bb, seed=bb + 2)
    got = gpu_frob(a, ab, b, bb)
    assert np.array_equal(got, O.frob_mul(a, ab, b, bb))
    assert np.array_equal(gpu_frob(b, bb, a, ab), got)


def test_frob_mul_edge_cases():
    a = operand(700, seed=3)
    assert not gpu_frob(a, 700, np.zeros(1, np.uint64), 0).any()
    one = np.array([1], dtype=np.uint64)
    c = gpu_frob(a, 700, one, 1)
    assert np.array_equal(c[:len(a)], a) and not c[len(a):].any()
    noisy = a.copy()
    noisy[-1] |= np.uint64(0xF) << np.uint64(60)   # bits above a_bits are ignored
    assert np.array_equal(gpu_frob(noisy, 700, a, 700), gpu_frob(a, 700, a, 700))


@pytest.mark.parametrize("bits", [1 << 20, (1 << 22) + 64])
def test_frob_mul_large_vs_alg5(bits):
    a, b = operand_pair(bits, seed=31)
    got = gpu_frob(a, bits, b, bits)
    assert np.array_equal(got, host(G.gf2x_mul(dev(a), bits, dev(b), bits)))
    if bits == 1 << 20:
        assert np.array_equal(got, O.mul_karatsuba(a, b))


def test_frob_mul_c4a_sampled_and_timing():
    # BASELINE's 2^28-bit size: sampled output words by the oracle one at a time, the mod-p check, and the time
    bits = 1 << 28
    a, b = operand_pair(bits, seed=5)
    da, db = dev(a), dev(b)
    c = G.gf2x_mul_frob(da, bits, db, bits)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.gf2x_mul_frob(da, bits, db, bits, c)
    e1.record()
    torch.cuda.synchronize()
    print(f"App. C multiply, 2^28-bit operands: {e0.elapsed_time(e1):.2f} ms")
    got = host(c)
    rng = np.random.default_rng(3)
    for w in sorted({0, 1, len(got) // 2, len(got) - 2, len(got) - 1} | set(int(x) for x in rng.integers(0, len(got), 10))):
        assert int(got[w]) == O.mul_word(a, b, w), w
    assert O.check_mod_p(a, b, got, O.random_irreducibles(3, seed=17))


_SWEEPS_ONLY = r"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1708_09746_b200 as G
from gf2x_synth import operand
M = int(sys.argv[1])
f = operand(1 << M, seed=M + 500)
d = torch.from_numpy(f.view(np.int64).copy()).cuda().view(torch.uint64)
G.gf2x_basis_cvt_bits(d, M)
torch.cuda.synchronize()
np.save(sys.argv[2], d.cpu().view(torch.int64).numpy())
"""


@pytest.mark.parametrize("env", ["GF2X_BITCVT_SWEEPS", "GF2X_BITCVT_NOCHUNK", "GF2X_BITCVT_NOREG"])
@pytest.mark.parametrize("M", [9, 20])
def test_bit_basis_cvt_sweeps_only_variant(M, env, tmp_path):
    # GF2X_BITCVT_SWEEPS=1: no word-level passes; GF2X_BITCVT_NOCHUNK=1: no shared-memory chunk pass;
    # GF2X_BITCVT_NOREG=1: 2^16-bit chunks with every step swept (no register passes); same result
    import os
    import subprocess
    import sys
    out = tmp_path / "g.npy"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", _SWEEPS_ONLY, str(M), str(out)], cwd=root, check=True, timeout=600,
                   env={**os.environ, env: "1"})
    f = operand(1 << M, seed=M + 500)
    assert np.array_equal(np.load(out).view(np.uint64), O.basis_cvt_bits(f, M))
