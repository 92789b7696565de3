"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bar: integer/bit work, so every product word must be bit-exact.  Small and
medium sizes are compared element by element with the oracle (brute force / Karatsuba / the paper's
Alg. 5); the BASELINE.json full sizes (2^28, 2^29 bits) in the launch configuration bench.py times
are checked on sampled output words the oracle computes one by one (O(n) each), by the product modulo
random irreducible degree-64 polynomials, and by the squaring closed form.
"""
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


def gpu_mul(a, ab, b, bb):
    return host(G.gf2x_mul(dev(a), ab, dev(b), bb))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1708_09746_b200 import build
    build.build()
    G.load()


# ------------------------------------------------------------------ small / ragged / edge cases
@pytest.mark.parametrize("bits", [1, 2, 31, 63, 64, 65, 100, 127, 128, 129, 191, 192, 193, 255, 256, 257,
                                  1000, 2047, 2048, 2049, 4095, 4097, 64 * 33, 64 * 63 + 5, 64 * 64 + 1])
def test_square_sizes_vs_brute(bits):
    a, b = operand_pair(bits, seed=1000 + bits)
    assert np.array_equal(gpu_mul(a, bits, b, bits), brute_mul_words(a, b))


@pytest.mark.parametrize("ab,bb", [(1, 1), (1, 64 * 50), (64 * 50, 1), (64, 65), (64 * 7 + 3, 128), (5000, 130),
                                   (64, 64 * 64 + 1), (3, 2), (64 * 1024, 64 * 3), (64 * 3, 64 * 1024 + 17)])
def test_unequal_sizes_vs_brute(ab, bb):
    a, b = operand(ab, seed=ab), operand(bb, seed=bb + 7)
    got = gpu_mul(a, ab, b, bb)
    assert np.array_equal(got, brute_mul_words(a, b))
    assert np.array_equal(gpu_mul(b, bb, a, ab), got)  # commutativity


def test_zero_length_one_and_zero():
    a = operand(300)
    z = gpu_mul(a, 300, np.zeros(1, np.uint64), 0)
    assert len(z) == 5 and not z.any()
    one = np.array([1], dtype=np.uint64)
    r = gpu_mul(a, 300, one, 1)
    assert np.array_equal(r[: len(a)], a) and not r[len(a):].any()
    assert not gpu_mul(a, 300, np.zeros(1, np.uint64), 1).any()


def test_bits_above_length_ignored():
    a, b = operand_pair(1000)
    dirty = a.copy()
    dirty[-1] |= np.uint64(0xFFFFFF << 40)   # 1000 bits = 15 words + 40 bits
    assert np.array_equal(gpu_mul(dirty, 1000, b, 1000), gpu_mul(a, 1000, b, 1000))


def test_shift_and_square_closed_forms():
    bits = 1 << 16
    a = operand(bits, seed=77)
    assert np.array_equal(gpu_mul(a, bits, a, bits), square_closed_form(a))
    for k in [0, 1, 63, 64, 4097, bits - 1]:
        xk = np.zeros(bits // 64, dtype=np.uint64)
        xk[k // 64] = np.uint64(1 << (k % 64))
        assert np.array_equal(gpu_mul(a, bits, xk, bits), brute_mul_words(a, xk))


def test_aliasing_rejected():
    a = dev(operand(640))
    with pytest.raises(G.Gf2xError, match="EINVAL"):
        G.gf2x_mul(a, 640, a, 640, c=a)


# ------------------------------------------------------------------ stage-level parity (R9 rule)
@pytest.mark.parametrize("bits", [64 * 8, 1 << 14, 1 << 18, 1 << 20, 1 << 22, 1 << 23])
def test_stage_intermediates_match_oracle(bits):
    a, b = operand_pair(bits, seed=5)
    _, st = O.alg5_mul(a, bits, b, bits, stages=True)
    names = {1: "cvt_a", 2: "fft_a", 3: "prod", 4: "ifft", 5: "icvt"}
    da, db = dev(a), dev(b)
    for s, nm in names.items():
        got = host(G.gf2x_debug_stage(da, bits, db, bits, s)).reshape(-1, 2)
        assert np.array_equal(got, st[nm]), f"stage {s} ({nm})"


# ------------------------------------------------------------------ BASELINE configs
def test_c1_exact():
    bits, _ = CONFIGS["c1"]
    a, b = operand_pair(bits)
    got = gpu_mul(a, bits, b, bits)
    assert np.array_equal(got, brute_mul_words(a, b))
    assert np.array_equal(got, O.alg5_mul(a, bits, b, bits))


def test_c2_batched_exact():
    bits, count = CONFIGS["c2"]
    A, B = batch_pair(bits, count)
    want = [O.mul_karatsuba(A[i], B[i]) for i in range(count)]
    dA, dB = dev(A), dev(B)
    for rep in range(4):   # repeated: a shared-memory race shows up as an intermittent mismatch
        C = host(G.gf2x_mul_batched(dA, bits, dB, bits, count))
        assert C.shape == (count, 2 * (bits // 64))
        bad = [i for i in range(count) if not np.array_equal(C[i], want[i])]
        assert not bad, (rep, bad[:10])


@pytest.mark.parametrize("ab,bb,count", [(1 << 22, 1 << 22, 3), (1 << 23, (1 << 21) + 77, 1), ((1 << 22) - 5, 1 << 23, 1)])
def test_residue_class_conversion_sizes(ab, bb, count):
    # sizes whose top Taylor steps (K = 16) run as residue-class passes (k_cvt_res), batched and unequal
    A, B = batch_pair(ab, count, seed=ab ^ bb) if ab == bb else (operand(ab, seed=1)[None], operand(bb, seed=2)[None])
    if ab == bb:
        C = host(G.gf2x_mul_batched(dev(A), ab, dev(B), bb, count))
    else:
        C = gpu_mul(A[0], ab, B[0], bb)[None]
    for i in range(count):
        want = O.mul_karatsuba(A[i], B[i]) if ab == bb else O.alg5_mul(A[i], ab, B[i], bb)
        assert np.array_equal(C[i], want), i


def test_batched_ragged_sizes():
    for bits, count in [(1, 5), (65, 33), (64 * 3 + 1, 17), (1000, 7), (64 * 64 + 1, 3)]:
        A, B = batch_pair(bits, count, seed=bits)
        C = host(G.gf2x_mul_batched(dev(A), bits, dev(B), bits, count))
        for i in range(count):
            assert np.array_equal(C[i], brute_mul_words(A[i], B[i]))


def test_c3_exact():
    bits, _ = CONFIGS["c3"]
    a, b = operand_pair(bits)
    got = gpu_mul(a, bits, b, bits)
    assert np.array_equal(got, O.mul_karatsuba(a, b))


def _sampled_words(n_out, rng, k=48):
    idx = {0, 1, 2, n_out // 2 - 1, n_out // 2, n_out // 2 + 1, n_out - 3, n_out - 2, n_out - 1}
    idx |= set(int(x) for x in rng.integers(0, n_out, size=k))
    return sorted(idx)


@pytest.mark.parametrize("cfg", ["c4a", "c4b"])
def test_full_size_sampled_words_and_mod_p(cfg):
    # the launch configuration bench.py times: one gf2x_mul on device-resident operands
    bits, _ = CONFIGS[cfg]
    a, b = operand_pair(bits)
    got = gpu_mul(a, bits, b, bits)
    n = len(a)
    assert got.shape == (2 * n,)
    rng = np.random.default_rng(7)
    for w in _sampled_words(2 * n, rng):
        assert int(got[w]) == O.mul_word(a, b, w), w
    assert not got[-1] >> np.uint64(63)  # degree 2*bits-2 < 2*bits-1
    assert O.check_mod_p(a, b, got, O.random_irreducibles(4, seed=zlib.crc32(cfg.encode()) & 0xFFFF))


def test_c4a_square_closed_form():
    bits, _ = CONFIGS["c4a"]
    a = operand(bits, seed=3)
    assert np.array_equal(gpu_mul(a, bits, a, bits), square_closed_form(a))


def test_workspace_api_matches_default_path():
    bits = 1 << 18
    a, b = operand_pair(bits, seed=2)
    nbytes = G.gf2x_workspace_bytes(bits, bits, 1)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    c = torch.empty(2 * len(a), dtype=torch.uint64, device="cuda")
    G.gf2x_mul_ws(dev(a), bits, dev(b), bits, c, 1, ws)
    assert np.array_equal(host(c), gpu_mul(a, bits, b, bits))
    small = torch.empty(nbytes // 2, dtype=torch.uint8, device="cuda")
    with pytest.raises(G.Gf2xError, match="ENOMEM"):
        G.gf2x_mul_ws(dev(a), bits, dev(b), bits, c, 1, small)


def test_stream_ordering_on_side_stream():
    bits = 1 << 16
    a, b = operand_pair(bits, seed=11)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        da, db = dev(a), dev(b)
        c = G.gf2x_mul(da, bits, db, bits, stream=s)
    s.synchronize()
    assert np.array_equal(host(c), brute_mul_words(a, b))


# ------------------------------------------------------------------ multi-GPU decomposition (one device)
@pytest.mark.parametrize("bits,ranks", [(1 << 22, 2), (1 << 23, 4), (1 << 24, 8), (1 << 24, 2)])
def test_sharded_simulation_exact(bits, ranks):
    # the partitioned FFT of SURVEY §8(e) with `ranks` virtual ranks: exchanges as peer-memory pulls (the
    # fused pull-pack / pull-unpack all-to-all kernels read the other ranks' buffers) and, with
    # GF2X_SHARD_LISTS=1, as the transfer lists the NCCL fallback sends (device copies)
    import os
    a, b = operand_pair(bits, seed=bits + ranks)
    want = O.mul_karatsuba(a, b)
    got = host(G.gf2x_mul_sharded_sim(dev(a), dev(b), bits, ranks))
    assert np.array_equal(got, want)
    os.environ["GF2X_SHARD_LISTS"] = "1"
    try:
        got = host(G.gf2x_mul_sharded_sim(dev(a), dev(b), bits, ranks))
    finally:
        del os.environ["GF2X_SHARD_LISTS"]
    assert np.array_equal(got, want)


def test_sharded_simulation_stages_match_oracle():
    bits = 1 << 23
    a, b = operand_pair(bits, seed=9)
    _, st = O.alg5_mul(a, bits, b, bits, stages=True)
    for ranks in (2, 4):
        for stage, key in ((1, "fft_a"), (5, "icvt")):
            got = host(G.gf2x_debug_shard_stage(dev(a), dev(b), bits, ranks, stage)).reshape(-1, 2)
            assert np.array_equal(got, st[key]), (ranks, stage)


# ------------------------------------------------------------------ c5: 2^32-bit operands (BASELINE configs[4])
@pytest.fixture(scope="module")
def c5_product():
    bits, _ = CONFIGS["c5"]
    a, b = operand_pair(bits)
    da, db = dev(a), dev(b)
    c = G.gf2x_mul(da, bits, db, bits)
    torch.cuda.synchronize()
    return bits, a, b, da, db, c


def test_c5_single_gpu_sampled_words_and_mod_p(c5_product):
    bits, a, b, _, _, c = c5_product
    got = host(c)
    n = len(a)
    rng = np.random.default_rng(11)
    for w in sorted({0, n - 1, n, 2 * n - 1} | set(int(x) for x in rng.integers(0, 2 * n, size=4))):
        assert int(got[w]) == O.mul_word(a, b, w), w
    assert not got[-1] >> np.uint64(63)
    assert O.check_mod_p(a, b, got, O.random_irreducibles(2, seed=5))


def test_c5_sharded_decomposition_8_ranks(c5_product):
    # the configuration bench.py --gpus 8 runs (8 ranks, NCCL exchanges), here as 8 virtual ranks on one
    # device: identical to the single-GPU product word for word
    bits, _, _, da, db, c = c5_product
    got = G.gf2x_mul_sharded_sim(da, db, bits, 8)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int64), c.view(torch.int64))
