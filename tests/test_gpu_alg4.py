"""GPU parity of Alg. 4 (sec 3.1) through the C ABI against the oracle:
products vs brute force / Karatsuba / sampled words, FFT and pointmul stages vs the oracle's Alg. 4."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from oracle.brute import brute_mul_words  # noqa: E402
from gf2x_synth import CONFIGS, batch_pair, operand, operand_pair  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def mul(a, ab, b, bb, batch=1):
    return host(G.gf2x_mul_alg4(dev(a), ab, dev(b), bb, batch=batch)).reshape(batch, -1)


@pytest.mark.parametrize("bits", [1, 2, 63, 64, 65, 128, 129, 1000, 2048, 4097, 64 * 64 + 1])
def test_sizes_vs_brute(bits):
    a, b = operand_pair(bits, seed=3000 + bits)
    assert np.array_equal(mul(a, bits, b, bits)[0], brute_mul_words(a, b))


def test_unequal_and_batched():
    for ab, bb in [(1, 64 * 50), (64 * 7 + 3, 128), (5000, 130), (64 * 1024, 64 * 3)]:
        a, b = operand(ab, seed=ab), operand(bb, seed=bb + 9)
        assert np.array_equal(mul(a, ab, b, bb)[0], brute_mul_words(a, b))
    A, B = batch_pair(1 << 12, 9, seed=5)
    C = mul(A, 1 << 12, B, 1 << 12, batch=9)
    for k in range(9):
        assert np.array_equal(C[k], O.mul_karatsuba(A[k], B[k]))


@pytest.mark.parametrize("bits", [64 * 8, 1 << 14, 1 << 18])
def test_stages_match_oracle(bits):
    a, b = operand_pair(bits, seed=33)
    _, st = O.alg4_mul(a, bits, b, bits, stages=True)
    da, db = dev(a), dev(b)
    for s, nm in {2: "fft_a", 3: "prod"}.items():
        got = host(G.gf2x_debug_stage_alg4(da, bits, db, bits, s)).reshape(-1, 2)
        assert np.array_equal(got, st[nm]), (s, nm)


def test_c3_exact():
    bits, _ = CONFIGS["c3"]
    a, b = operand_pair(bits)
    assert np.array_equal(mul(a, bits, b, bits)[0], O.mul_karatsuba(a, b))


def test_c4a_sampled_words():
    bits, _ = CONFIGS["c4a"]
    a, b = operand_pair(bits)
    got = mul(a, bits, b, bits)[0]
    n = len(a)
    rng = np.random.default_rng(21)
    for w in sorted({0, n - 1, n, 2 * n - 1} | set(int(x) for x in rng.integers(0, 2 * n, size=12))):
        assert int(got[w]) == O.mul_word(a, b, w), w
    assert O.check_mod_p(a, b, got, O.random_irreducibles(2, seed=44))
