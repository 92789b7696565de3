"""Full-size element-wise parity: every output word of the CUDA product at the sizes
bench.py times (c4a, c4b, and the single-GPU c5) against the oracle's product, through SHA-256 digests
of all n_a + n_b words.  The digests in tests/golden/oracle_digests.json were written by
tools/make_digests.py, which calls only oracle/ (the paper's Alg. 5 step by step) on the gf2x_synth
seeded operands -- no value there comes from the CUDA path.  Launch configuration: one gf2x_mul on
device-resident operands, exactly as bench.py's timed step."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import CONFIGS, DEFAULT_SEED, operand_pair  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_digests.json")))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1708_09746_b200 import build
    build.build()
    G.load()


@pytest.mark.parametrize("cfg", ["c3", "c4a", "c4b", "c5"])
def test_full_product_digest(cfg):
    g = GOLD["digests"][cfg]
    bits, _ = CONFIGS[cfg]
    assert g["bits"] == bits and GOLD["seed"] == DEFAULT_SEED
    a, b = operand_pair(bits, DEFAULT_SEED)
    da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
    del a, b
    c = G.gf2x_mul(da, bits, db, bits)
    torch.cuda.synchronize()
    del da, db
    got = c.cpu().view(torch.int64).numpy().view(np.uint64)
    del c
    assert len(got) == g["words"]
    assert f"0x{int(got[0]):016x}" == g["first_word"] and f"0x{int(got[-1]):016x}" == g["last_word"]
    assert hashlib.sha256(got.astype("<u8").tobytes()).hexdigest() == g["sha256"]
