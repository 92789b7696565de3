"""The digest fixture's procedure pinned against an independent algorithm (no GPU): for c3 the oracle's
Alg. 5 product digest stored in tests/golden/oracle_digests.json equals the SHA-256 of the O2 Karatsuba
product (a different algorithm on the same seeded operands), so a digest mismatch on the GPU cannot come
from the way the fixture was written."""
import hashlib
import json
import os

import numpy as np

import oracle as O
from gf2x_synth import CONFIGS, DEFAULT_SEED, operand_pair

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_digests.json")))


def test_c3_digest_is_the_karatsuba_product():
    bits, _ = CONFIGS["c3"]
    a, b = operand_pair(bits, DEFAULT_SEED)
    c = O.mul_karatsuba(a, b)
    g = GOLD["digests"]["c3"]
    assert g["words"] == len(c) and g["bits"] == bits
    assert hashlib.sha256(c.astype("<u8").tobytes()).hexdigest() == g["sha256"]


def test_digest_fixture_covers_bench_sizes():
    for cfg in ("c4a", "c4b", "c5"):
        g = GOLD["digests"].get(cfg)
        assert g is not None, cfg
        assert g["bits"] == CONFIGS[cfg][0] and g["words"] == 2 * ((g["bits"] + 63) // 64)
        assert len(g["sha256"]) == 64 and int(g["sha256"], 16) >= 0
