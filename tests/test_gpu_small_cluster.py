"""GPU parity of the fused small-product kernel k_small (csrc/small.cuh) in each cluster shape, against the
oracle's Karatsuba on the same seeded operands: CL = 4 (one limb per CTA), 8 (limbs x two point segments:
the top FFT layer crosses CTAs) and 16 (limbs x four segments: the top two layers, with the GF(4) multiplier
s_(m-2)(v_(m-1)), cross CTAs; iBasisCvt gathers each limb whole).  GF2X_SMALL_CL caps the cluster (read per
call).  Products of N = 2^7 .. 2^11 points, equal, unequal and ragged operands."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import operand  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1708_09746_b200 import build
    build.build()
    G.load()


def ref(a, b):
    n = max(len(a), len(b))
    pa, pb = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    pa[: len(a)], pb[: len(b)] = a, b
    return O.mul_karatsuba(pa, pb)[: len(a) + len(b)]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


# (a_bits, b_bits): m = ceil(log2(na + nb)) = 7, 8, 9, 10, 11 and ragged / unequal shapes
SHAPES = [(4000, 4096), (6000, 6000), (9000, 7777), (20000, 20001), (1 << 16, 1 << 16), ((1 << 16) - 13, 3000),
          (64 * 1000 + 1, 64 * 23 + 5), (1 << 15, (1 << 15) + 1)]


@pytest.mark.parametrize("cl", ["4", "8", "16"])
@pytest.mark.parametrize("knobs", [{}, {"GF2X_SMALL_NO_SEGCVT": "1"}, {"GF2X_SMALL_NO_KT": "1"}])
def test_small_cluster_shapes_exact(cl, knobs, monkeypatch):
    """(knobs: segment-local conversions off; precomputed FFT constants off)"""
    monkeypatch.setenv("GF2X_SMALL_CL", cl)
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    for ab, bb in SHAPES:
        a, b = operand(ab, seed=ab + 3), operand(bb, seed=bb + 11)
        G.profile_enable(True)
        got = G.gf2x_mul(dev(a), ab, dev(b), bb)
        torch.cuda.synchronize()
        kern = {r["kernel"] for r in G.profile_report()}
        G.profile_enable(False)
        got = got.cpu().view(torch.int64).numpy().view(np.uint64)
        assert np.array_equal(got, ref(a, b)), (cl, ab, bb)
        assert len(kern) == 1 and next(iter(kern)).startswith("k_small<"), kern
        m = int(np.ceil(np.log2((ab + 63) // 64 + (bb + 63) // 64)))
        want = 16 if (cl == "16" and m >= 9) else (8 if (cl in ("8", "16") and m >= 8) else 4)
        # (a device that cannot hold a 16-CTA cluster runs 8)
        assert next(iter(kern)) in ({f"k_small<{want}>", "k_small<8>"} if want == 16 else {f"k_small<{want}>"}), kern


def test_small_cluster_repeated_c1_shape(monkeypatch):
    """The c1 shape ten times in a row on one stream (the cluster barriers order the DSMEM reads and writes;
    a race would show up as a differing product)."""
    monkeypatch.delenv("GF2X_SMALL_CL", raising=False)
    bits = 1 << 16
    a, b = operand(bits, seed=5), operand(bits, seed=6)
    want = O.mul_karatsuba(a, b)
    da, db = dev(a), dev(b)
    outs = [G.gf2x_mul(da, bits, db, bits) for _ in range(10)]
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().view(torch.int64).numpy().view(np.uint64), want)


@pytest.mark.parametrize("bits,count", [(9000, 37), (1 << 14, 300), (2000, 5)])
def test_small_batch_mode_exact(bits, count, monkeypatch):
    """GF2X_SMALL_BATCH=1: one persistent CTA per product (k_small<1>, all four limbs, the FFT constants
    precomputed once per CTA and reused by every product it takes) against Karatsuba, every product."""
    from gf2x_synth import batch_pair
    monkeypatch.setenv("GF2X_SMALL_BATCH", "1")
    a, b = batch_pair(bits, count, seed=bits)
    G.profile_enable(True)
    got = G.gf2x_mul_batched(dev(a.reshape(-1)), bits, dev(b.reshape(-1)), bits, count)
    torch.cuda.synchronize()
    kern = {r["kernel"] for r in G.profile_report()}
    G.profile_enable(False)
    assert kern == {"k_small<1>"}, kern
    got = got.cpu().view(torch.int64).numpy().view(np.uint64).reshape(count, -1)
    for i in range(count):
        assert np.array_equal(got[i], O.mul_karatsuba(a[i], b[i])), i
