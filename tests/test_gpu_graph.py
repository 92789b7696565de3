"""CUDA-graph capture of the multiply (the library's launches are stream-ordered, host planning happens at
capture time, and the truncated path's side stream forks / joins by events): capture once on a stream,
replay with new operands copied into the static buffers, compare with the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from oracle.brute import brute_mul_words  # noqa: E402
from gf2x_synth import batch_pair, operand  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def capture(fn, s):
    with torch.cuda.stream(s):
        for _ in range(2):   # workspace and side stream for s exist before the capture
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    return g


@pytest.mark.parametrize("ab,bb", [(1 << 16, 1 << 16), (1000, 70000), ((1 << 23) + 192, (1 << 23) + 192)])
def test_capture_replay_single(ab, bb):
    s = torch.cuda.Stream()
    da, db = dev(operand(ab, seed=1)), dev(operand(bb, seed=2))
    dc = torch.empty(G.nwords(ab) + G.nwords(bb), dtype=torch.uint64, device="cuda")
    g = capture(lambda: G.gf2x_mul(da, ab, db, bb, dc, stream=s), s)
    for seed in (11, 12, 13):
        a, b = operand(ab, seed=seed), operand(bb, seed=seed + 100)
        da.copy_(dev(a))
        db.copy_(dev(b))
        with torch.cuda.stream(s):
            g.replay()
        want = O.alg5_mul(a, ab, b, bb) if max(ab, bb) > 1 << 17 else brute_mul_words(a, b)
        assert np.array_equal(host(dc), want), seed


def test_capture_replay_batched_and_w128():
    s = torch.cuda.Stream()
    bits, count = 1 << 14, 64
    A, B = batch_pair(bits, count, seed=5)
    da, db = dev(A.reshape(-1)), dev(B.reshape(-1))
    dc = torch.empty(count, 2 * G.nwords(bits), dtype=torch.uint64, device="cuda")
    dw = torch.empty(1, 2 * G.nwords(1 << 16), dtype=torch.uint64, device="cuda")
    wa, wb = dev(operand(1 << 16, seed=7)), dev(operand(1 << 16, seed=8))

    def both():
        G.gf2x_mul_batched(da, bits, db, bits, count, dc, stream=s)
        G.gf2x_mul_w(wa, 1 << 16, wb, 1 << 16, 128, 1, dw, stream=s)

    g = capture(both, s)
    A2, B2 = batch_pair(bits, count, seed=6)
    da.copy_(dev(A2.reshape(-1)))
    db.copy_(dev(B2.reshape(-1)))
    a2, b2 = operand(1 << 16, seed=9), operand(1 << 16, seed=10)
    wa.copy_(dev(a2))
    wb.copy_(dev(b2))
    with torch.cuda.stream(s):
        g.replay()
    C = host(dc).reshape(count, -1)
    for i in range(0, count, 7):
        assert np.array_equal(C[i], O.mul_karatsuba(A2[i], B2[i])), i
    assert np.array_equal(host(dw)[0], O.mul_karatsuba(a2, b2))


@pytest.mark.parametrize("ab,bb", [(20000, 20001), (5000, 3000)])
def test_capture_small_product_without_warmup(ab, bb):
    """A fused small product (k_small) captured on its very first call: the per-device constant table is not
    allocated during a capture (the kernel then builds its own), so the capture works either way."""
    s = torch.cuda.Stream()
    da, db = dev(operand(ab, seed=3)), dev(operand(bb, seed=4))
    dc = torch.empty(G.nwords(ab) + G.nwords(bb), dtype=torch.uint64, device="cuda")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        G.gf2x_mul(da, ab, db, bb, dc, stream=s)
    for seed in (21, 22):
        a, b = operand(ab, seed=seed), operand(bb, seed=seed + 100)
        da.copy_(dev(a))
        db.copy_(dev(b))
        with torch.cuda.stream(s):
            g.replay()
        assert np.array_equal(host(dc), brute_mul_words(a, b)), seed
