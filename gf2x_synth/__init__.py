"""Seeded synthetic operands for GF(2)[x] multiplication (shared by tests, bench and smoke).

This module holds NO arithmetic of the method -- only the input recipe:

* words are drawn from a counter-based SplitMix64 stream (Steele, Lea, Flood 2014):
  word i of stream `seed` is mix64(seed + (i + 1) * 0x9E3779B97F4A7C15);
* operand a uses seed S, operand b uses seed S + 1 (S defaults to 0x170809746);
* bits at positions >= `bits` are cleared and bit `bits - 1` is set, so the degree is exactly
  bits - 1 (BASELINE.json config 1 "leading bit forced 1"; the other configs follow the same rule);
* a batch of `count` operands of `bits` bits each is one stream, operand j occupying words
  [j * n, (j + 1) * n) with n = ceil(bits / 64); each operand is masked / top-bit-set individually.

Polynomial packing (§2.1): little-endian 64-bit words, bit i of
word j is the coefficient of x^(64 j + i).
"""
from __future__ import annotations

import numpy as np

DEFAULT_SEED = 0x170809746
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Words start .. start+count-1 of the counter-based SplitMix64 stream `seed` (uint64 array)."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def nwords(bits: int) -> int:
    return (bits + 63) // 64


def mask_operand(words: np.ndarray, bits: int, top_bit: bool = True) -> np.ndarray:
    """Clear bits >= `bits` and (optionally) set bit bits-1, in place on a 1-D or 2-D (batch) array."""
    n = nwords(bits)
    assert words.shape[-1] == n
    if bits == 0:
        return words
    r = bits - 64 * (n - 1)  # valid bits in the last word, 1..64
    if r < 64:
        words[..., n - 1] &= np.uint64((1 << r) - 1)
    if top_bit:
        words[..., n - 1] |= np.uint64(1 << (r - 1))
    return words


def operand(bits: int, seed: int = DEFAULT_SEED, top_bit: bool = True) -> np.ndarray:
    """One uniformly random polynomial of `bits` bits (degree bits-1 when top_bit)."""
    w = splitmix64(seed, nwords(bits))
    return mask_operand(w, bits, top_bit)


def operand_pair(bits: int, seed: int = DEFAULT_SEED, top_bit: bool = True):
    """(a, b) for one multiply: a from seed S, b from seed S+1."""
    return operand(bits, seed, top_bit), operand(bits, seed + 1, top_bit)


def batch(bits: int, count: int, seed: int = DEFAULT_SEED, top_bit: bool = True) -> np.ndarray:
    """`count` operands of `bits` bits, contiguous in one stream -> array of shape (count, n)."""
    n = nwords(bits)
    w = splitmix64(seed, n * count).reshape(count, n)
    return mask_operand(w, bits, top_bit)


def batch_pair(bits: int, count: int, seed: int = DEFAULT_SEED, top_bit: bool = True):
    return batch(bits, count, seed, top_bit), batch(bits, count, seed + 1, top_bit)


# BASELINE.json "configs" as (name, operand bits, batch) -- shapes only, no arithmetic.
CONFIGS = {
    "c1": (1 << 16, 1),      # single 2^16-bit multiply
    "c2": (1 << 14, 4096),   # 4096 independent 2^14-bit pairs
    "c3": (1 << 24, 1),      # single 2^24-bit multiply (FFT over 2^19 points)
    "c4a": (1 << 28, 1),     # paper headline 2^28-bit operands
    "c4b": (1 << 29, 1),     # paper headline 2^29-bit operands
    "c5": (1 << 32, 1),      # 2^32-bit operands, sharded across GPUs
}
