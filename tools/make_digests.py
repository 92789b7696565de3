#!/usr/bin/env python
"""Write tests/golden/oracle_digests.json: SHA-256 of the exact products of the seeded full-size
configs, computed by the CPU oracle alone (oracle/, the paper's Alg. 5 step by step, OpenMP).

SURVEY.md §8(d) ("cache the oracle's product digest ... as a test fixture"): the GPU parity tests
(tests/test_gpu_digests.py) compare the digest of every output word of the CUDA product at the
sizes bench.py times against these values.  This script imports only `oracle` and `gf2x_synth`
(the seeded input recipe); nothing here comes from the CUDA path.

    python tools/make_digests.py [c4a c4b c5 ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from gf2x_synth import CONFIGS, DEFAULT_SEED, operand_pair  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_digests.json")


def digest(words) -> str:
    return hashlib.sha256(words.astype("<u8").tobytes()).hexdigest()


def main(names):
    O.build()
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "source": "tools/make_digests.py: oracle/ Alg. 5 (or_alg5_mul) on the gf2x_synth seeded operands; "
                  "SHA-256 of the n_a + n_b little-endian uint64 product words",
        "seed": DEFAULT_SEED, "digests": {}}
    for name in names:
        bits, batch = CONFIGS[name]
        assert batch == 1, "digests are for single products"
        a, b = operand_pair(bits, DEFAULT_SEED)
        t0 = time.perf_counter()
        c = O.alg5_mul(a, bits, b, bits)
        dt = time.perf_counter() - t0
        assert len(c) == 2 * len(a)
        data["digests"][name] = {"bits": bits, "words": int(len(c)), "sha256": digest(c),
                                 "first_word": f"0x{int(c[0]):016x}", "last_word": f"0x{int(c[-1]):016x}",
                                 "oracle_s": round(dt, 1), "threads": O.num_threads()}
        print(name, data["digests"][name], flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c4a", "c4b", "c5"])
