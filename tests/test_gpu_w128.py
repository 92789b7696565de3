"""GPU parity of the w = 128 variant (Alg. 5 over TGF(2^256)) through the
C ABI (gf2x_mul_w / gf2x_debug_stage_w128) against the CPU oracle (O.alg5_mul_w128, brute force,
Karatsuba, single-word products, mod-p checks).  Bit-exact, like the w = 64 path."""
import zlib
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from oracle.brute import brute_mul_words, square_closed_form  # noqa: E402
from gf2x_synth import CONFIGS, batch_pair, operand, operand_pair  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def gpu_mul(a, ab, b, bb, batch=1):
    return host(G.gf2x_mul_w(dev(a), ab, dev(b), bb, w=128, batch=batch)).reshape(batch, -1)


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1708_09746_b200 import build
    build.build()
    G.load()


@pytest.mark.parametrize("bits", [1, 2, 63, 64, 65, 127, 128, 129, 255, 256, 257, 383, 1000, 2048, 4097,
                                  128 * 33, 128 * 63 + 5, 128 * 64 + 1])
def test_square_sizes_vs_brute(bits):
    a, b = operand_pair(bits, seed=2000 + bits)
    assert np.array_equal(gpu_mul(a, bits, b, bits)[0], brute_mul_words(a, b))


@pytest.mark.parametrize("ab,bb", [(1, 1), (1, 128 * 50), (128 * 50, 1), (64, 65), (128 * 7 + 3, 256), (5000, 130),
                                   (128, 128 * 64 + 1), (3, 2), (128 * 1024, 128 * 3), (64 * 3, 128 * 1024 + 17)])
def test_unequal_sizes_vs_brute(ab, bb):
    a, b = operand(ab, seed=ab + 5), operand(bb, seed=bb + 11)
    got = gpu_mul(a, ab, b, bb)[0]
    assert np.array_equal(got, brute_mul_words(a, b))
    assert np.array_equal(gpu_mul(b, bb, a, ab)[0], got)


def test_edge_cases():
    a = operand(300, seed=3)
    assert not gpu_mul(a, 300, np.zeros(1, np.uint64), 0).any()
    one = np.array([1], dtype=np.uint64)
    r = gpu_mul(a, 300, one, 1)[0]
    assert np.array_equal(r[: len(a)], a) and not r[len(a):].any()
    dirty = a.copy()
    dirty[-1] |= np.uint64(0xFFFF << 44)
    assert np.array_equal(gpu_mul(dirty, 300, a, 300), gpu_mul(a, 300, a, 300))
    with pytest.raises(G.Gf2xError):
        G.gf2x_mul_w(dev(a), 300, dev(a), 300, w=96)


@pytest.mark.parametrize("bits", [128 * 8, 1 << 14, 1 << 18, 1 << 21])
def test_stage_intermediates_match_oracle(bits):
    a, b = operand_pair(bits, seed=15)
    _, st = O.alg5_mul_w128(a, bits, b, bits, stages=True)
    da, db = dev(a), dev(b)
    for s, nm in {1: "cvt_a", 2: "fft_a", 3: "prod", 5: "icvt"}.items():
        got = host(G.gf2x_debug_stage_w128(da, bits, db, bits, s)).reshape(-1, 4)
        assert np.array_equal(got, st[nm]), f"stage {s} ({nm})"


def test_batched_exact():
    for bits, count in [(1, 3), (129, 17), (1 << 14, 64), (128 * 5 + 1, 9)]:
        A, B = batch_pair(bits, count, seed=bits + 1)
        C = gpu_mul(A, bits, B, bits, batch=count)
        for i in range(count):
            assert np.array_equal(C[i], O.mul_karatsuba(A[i], B[i]) if bits % 64 == 0 else brute_mul_words(A[i], B[i])), i


def test_c2_batched_exact():
    bits, count = CONFIGS["c2"]
    A, B = batch_pair(bits, count)
    C = gpu_mul(A, bits, B, bits, batch=count)
    bad = [i for i in range(count) if not np.array_equal(C[i], O.mul_karatsuba(A[i], B[i]))]
    assert not bad, bad[:10]


def test_c3_exact_and_same_as_w64():
    bits, _ = CONFIGS["c3"]
    a, b = operand_pair(bits)
    got = gpu_mul(a, bits, b, bits)[0]
    assert np.array_equal(got, O.mul_karatsuba(a, b))
    assert np.array_equal(got, host(G.gf2x_mul(dev(a), bits, dev(b), bits)))


def _sampled_words(n_out, rng, k=48):
    idx = {0, 1, 2, n_out // 2 - 1, n_out // 2, n_out // 2 + 1, n_out - 3, n_out - 2, n_out - 1}
    idx |= set(int(x) for x in rng.integers(0, n_out, size=k))
    return sorted(idx)


@pytest.mark.parametrize("cfg", ["c4a", "c4b"])
def test_full_size_sampled_words_and_mod_p(cfg):
    bits, _ = CONFIGS[cfg]
    a, b = operand_pair(bits)
    got = gpu_mul(a, bits, b, bits)[0]
    n = len(a)
    rng = np.random.default_rng(11)
    for w in _sampled_words(2 * n, rng):
        assert int(got[w]) == O.mul_word(a, b, w), w
    assert O.check_mod_p(a, b, got, O.random_irreducibles(4, seed=(zlib.crc32(cfg.encode()) + 128) & 0xFFFF))


def test_c4a_square_closed_form():
    bits, _ = CONFIGS["c4a"]
    a = operand(bits, seed=8)
    assert np.array_equal(gpu_mul(a, bits, a, bits)[0], square_closed_form(a))
