"""GPU parity of the truncated FFT (trunc.cuh; R21): products whose L = n_a + n_b - 1
blocks lie just above a power of two run an H-point multiply plus a 2^j-point one instead of an N-point one.
The result is the exact product (oracle: Karatsuba / Alg. 5 / brute force / sampled words + mod p)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import operand  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


TRUNC_KERNELS = {"k_trunc_reduce", "k_trunc_fold"}   # fused Reduce passes / the layered debug path


def gpu_mul(a, ab, b, bb, profile=False):
    if profile:
        G.profile_enable(True)
    c = host(G.gf2x_mul(dev(a), ab, dev(b), bb))
    names = set()
    if profile:
        names = {r["kernel"] for r in G.profile_report()}
        G.profile_enable(False)
    return c, names


@pytest.mark.parametrize("ab,bb", [((1 << 20) + 64, (1 << 20) + 64), ((1 << 20) + 1, (1 << 20) + 65), (1 << 20, (1 << 20) + 3000),
                                   ((1 << 20) + 64 * 4095, (1 << 20) + 7), ((1 << 19) + 999, (1 << 21) - 64 * 100),
                                   ((1 << 22) + 1, (1 << 22) + 1),
                                   # one operand reaching past H (its tail joins the upper part unreduced)
                                   ((1 << 20) + 128, 3000), (3000, (1 << 20) + 128), ((1 << 20) + 64 * 4000, 64 * 90 - 5),
                                   ((1 << 22) + 64 * 3, 64 * 4000)])
def test_truncated_products_exact(ab, bb):
    a, b = operand(ab, seed=ab % 1000 + 1), operand(bb, seed=bb % 1000 + 2)
    got, names = gpu_mul(a, ab, b, bb, profile=True)
    assert names & TRUNC_KERNELS   # the truncated path ran
    assert np.array_equal(got, O.alg5_mul(a, ab, b, bb))


def test_not_truncated_when_not_eligible():
    ab = 1 << 20   # L = 2^15 - 1: exactly a power-of-two transform, nothing to truncate
    a, b = operand(ab, seed=1), operand(ab, seed=2)
    got, names = gpu_mul(a, ab, b, ab, profile=True)
    assert not names & TRUNC_KERNELS
    assert np.array_equal(got, O.mul_karatsuba(a, b))


def test_truncated_large_sampled_words_and_mod_p():
    ab = (1 << 28) + 64
    a, b = operand(ab, seed=5), operand(ab, seed=6)
    got, names = gpu_mul(a, ab, b, ab, profile=True)
    assert names & TRUNC_KERNELS
    n_out = len(got)
    rng = np.random.default_rng(9)
    for w in sorted({0, n_out // 2 - 1, n_out // 2, n_out - 3, n_out - 2, n_out - 1} |
                    set(int(x) for x in rng.integers(0, n_out, size=12))):
        assert int(got[w]) == O.mul_word(a, b, w), w
    assert O.check_mod_p(a, b, got, O.random_irreducibles(3, seed=31))


_VARIANT = r"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1708_09746_b200 as G
from gf2x_synth import operand
ab, bb = int(sys.argv[1]), int(sys.argv[2])
a, b = operand(ab, seed=71), operand(bb, seed=72)
da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
c = G.gf2x_mul(da, ab, db, bb)
torch.cuda.synchronize()
np.save(sys.argv[3], c.cpu().view(torch.int64).numpy())
"""


@pytest.mark.parametrize("env", ["GF2X_TRUNC_NOFUSE", "GF2X_TRUNC_SERIAL", "GF2X_TRUNC_LAYERED", "GF2X_NO_CVT_SPLIT"])
def test_truncated_variants_agree(env, tmp_path):
    # the debug / fallback variants of the truncated path (flags are read once per process: a subprocess each)
    import os
    import subprocess
    import sys
    ab = bb = (1 << 23) + 64 * 3   # m = 19: the fused Reduce applies (j = 12 = k_lo)
    a, b = operand(ab, seed=71), operand(bb, seed=72)
    want = O.alg5_mul(a, ab, b, bb)
    out = tmp_path / "c.npy"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", _VARIANT, str(ab), str(bb), str(out)], cwd=root, check=True, timeout=600,
                   env={**os.environ, env: "1"})
    assert np.array_equal(np.load(out).view(np.uint64), want)


@pytest.mark.parametrize("bits", [(1 << 23) + 192, (1 << 24) + 64, 1 << 20, ((1 << 16) + 5) * 64])
def test_launch_count_matches_profile(bits):
    # gf2x_launch_count (bench.py's gpu_launches claim) = the launches the profiler records for one multiply
    a, b = operand(bits, seed=3), operand(bits, seed=4)
    G.gf2x_mul(dev(a), bits, dev(b), bits)
    torch.cuda.synchronize()
    _, _ = gpu_mul(a, bits, b, bits, profile=False)
    G.profile_enable(True)
    G.gf2x_mul(dev(a), bits, dev(b), bits)
    torch.cuda.synchronize()
    n = sum(r["launches"] for r in G.profile_report())
    G.profile_enable(False)
    assert n == G.gf2x_launch_count(bits, bits)
