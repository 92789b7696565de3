"""GPU parity of both inverse tails (R28) against the oracle, in one process:
  * the default: changeRepr^-1 + the combine written in the novel basis (k_ipsi_bs<true> / k_ipsi256_bs<true>), then
    iBasisCvt of the combined words in place in a 16-byte aligned output;
  * an output only 8-byte aligned (a view one word into a buffer): the 128-bit (w = 64) / two-plane (w = 128)
    iBasisCvt, then changeRepr^-1 + InterleavedCombine, as Alg. 5 orders them.
Both must give the oracle's product word for word, and they must have run different kernels."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import batch_pair, operand_pair  # noqa: E402


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).reshape(-1).view(np.int64)).cuda().view(torch.uint64)


def _run(fn, n_out, aligned):
    buf = torch.zeros(n_out + 2, dtype=torch.uint64, device="cuda")
    c = buf[:n_out] if aligned else buf[1:n_out + 1]
    G.profile_enable(True)
    fn(c)
    torch.cuda.synchronize()
    kern = {r["kernel"] for r in G.profile_report()}
    G.profile_enable(False)
    return c.cpu().view(torch.int64).numpy().view(np.uint64).copy(), kern


@pytest.mark.parametrize("bits", [1 << 18, 1 << 21, (1 << 22) + (1 << 21)])
def test_alg5_both_tails(bits):
    a, b = operand_pair(bits, seed=bits % 89)
    want = O.alg5_mul(a, bits, b, bits)
    da, db = _dev(a), _dev(b)
    n = len(want)
    got_a, k_a = _run(lambda c: G.gf2x_mul(da, bits, db, bits, c), n, True)
    got_u, k_u = _run(lambda c: G.gf2x_mul(da, bits, db, bits, c), n, False)
    assert np.array_equal(got_a, want)
    assert np.array_equal(got_u, want)
    if bits & (bits - 1) == 0:   # the product fills all N words: the aligned output takes the R28 tail
        assert "k_ipsi_mcomb" in k_a and "k_ipsi_mcomb" not in k_u


def test_alg5_batched_both_tails():
    bits, batch = 1 << 14, 64
    a, b = batch_pair(bits, batch)
    want = np.stack([O.mul_karatsuba(a[i], b[i]) for i in range(batch)]).reshape(-1)
    da, db = _dev(a), _dev(b)
    got_a, k_a = _run(lambda c: G.gf2x_mul_batched(da, bits, db, bits, batch, c), len(want), True)
    got_u, k_u = _run(lambda c: G.gf2x_mul_batched(da, bits, db, bits, batch, c), len(want), False)
    assert np.array_equal(got_a, want) and np.array_equal(got_u, want)
    assert "k_ipsi_mcomb" in k_a and "k_ipsi_mcomb" not in k_u


@pytest.mark.parametrize("bits", [1 << 19, 1 << 22])
def test_w128_both_tails(bits):
    a, b = operand_pair(bits, seed=bits % 83)
    want = O.mul_karatsuba(a, b)
    da, db = _dev(a), _dev(b)
    got_a, k_a = _run(lambda c: G.gf2x_mul_w(da, bits, db, bits, 128, 1, c), len(want), True)
    got_u, k_u = _run(lambda c: G.gf2x_mul_w(da, bits, db, bits, 128, 1, c), len(want), False)
    assert np.array_equal(got_a, want) and np.array_equal(got_u, want)
    assert "k_ipsi256_mcomb" in k_a and "k_ipsi256_mcomb" not in k_u
