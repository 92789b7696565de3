"""Seeded random sweep of sizes through the C ABI (w = 64 and w = 128, single and batched) against the
oracle: unequal, ragged and power-of-two-boundary bit lengths up to 2^20 bits.  Bit-exact."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import batch_pair, operand  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def _sizes(seed, count):
    R = random.Random(seed)
    out = []
    for _ in range(count):
        kind = R.randrange(4)
        if kind == 0:   # around a power of two
            p = R.randrange(6, 21)
            a = (1 << p) + R.randrange(-70, 70)
        elif kind == 1:
            a = R.randrange(1, 1 << 12)
        else:
            a = R.randrange(1, 1 << 20)
        b = a if R.random() < 0.3 else max(1, int(a * R.uniform(0.01, 3.0)))
        out.append((max(1, a), min(b, 1 << 20)))
    return out


@pytest.mark.parametrize("w", [64, 128])
def test_random_sizes(w):
    for i, (ab, bb) in enumerate(_sizes(1708 + w, 60)):
        a, b = operand(ab, seed=3 * i + w), operand(bb, seed=3 * i + 1 + w)
        got = host(G.gf2x_mul_w(dev(a), ab, dev(b), bb, w=w)).reshape(-1)
        want = O.mul_schoolbook(a, b) if (ab + bb) < (1 << 15) else O.alg5_mul(a, ab, b, bb)
        assert np.array_equal(got, want), (w, ab, bb)


@pytest.mark.parametrize("w", [64, 128])
def test_random_batches(w):
    R = random.Random(99 + w)
    for i in range(12):
        bits = R.choice([R.randrange(1, 3000), 1 << R.randrange(8, 15), (1 << R.randrange(8, 14)) + R.randrange(1, 64)])
        count = R.randrange(1, 40)
        A, B = batch_pair(bits, count, seed=i + w)
        C = host(G.gf2x_mul_w(dev(A), bits, dev(B), bits, w=w, batch=count)).reshape(count, -1)
        for k in range(count):
            assert np.array_equal(C[k], O.mul_schoolbook(A[k], B[k])), (w, bits, count, k)
