"""A/B of k_small variants in one process (the knobs are read per call): c1 (or a given shape), CUDA events
over 200 back-to-back multiplies, variants interleaved over 7 rounds, median per variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_1708_09746_b200 as G
from gf2x_synth import operand_pair, batch_pair

VARIANTS = {
    "cl4": {"GF2X_SMALL_CL": "4"},
    "cl8": {"GF2X_SMALL_CL": "8"},
    "cl16": {"GF2X_SMALL_CL": "16"},
    "cl16_noseg": {"GF2X_SMALL_CL": "16", "GF2X_SMALL_NO_SEGCVT": "1"},
    "cl16_nokt": {"GF2X_SMALL_CL": "16", "GF2X_SMALL_NO_KT": "1"},
    "cl8_noseg": {"GF2X_SMALL_CL": "8", "GF2X_SMALL_NO_SEGCVT": "1"},
    "cl16_ktbuild": {"GF2X_SMALL_CL": "16", "GF2X_SMALL_KT_BUILD": "1"},
}
KNOBS = sorted({k for v in VARIANTS.values() for k in v})
bits = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if batch == 1:
    a, b = operand_pair(bits)
else:
    a, b = batch_pair(bits, batch)
    VARIANTS = {"batch_small": {"GF2X_SMALL_BATCH": "1"}, "batch_small_nokt": {"GF2X_SMALL_BATCH": "1", "GF2X_SMALL_NO_KT": "1"},
                "batch_small_ktbuild": {"GF2X_SMALL_BATCH": "1", "GF2X_SMALL_KT_BUILD": "1"},
                "multipass": {}}
    KNOBS = sorted({k for v in VARIANTS.values() for k in v})
da = torch.from_numpy(a.reshape(-1).view(np.int64)).cuda().view(torch.uint64)
db = torch.from_numpy(b.reshape(-1).view(np.int64)).cuda().view(torch.uint64)


def run():
    return G.gf2x_mul(da, bits, db, bits) if batch == 1 else G.gf2x_mul_batched(da, bits, db, bits, batch)


ref = run()
torch.cuda.synchronize()
res = {k: [] for k in VARIANTS}
reps = 200 if batch == 1 else 20
for rnd in range(7):
    for name, env in VARIANTS.items():
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.update(env)
        out = run()
        torch.cuda.synchronize()
        assert torch.equal(out, ref), name
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / reps * 1000)
for name, v in res.items():
    print(f"{name:18s} median {np.median(v):8.2f} us  min {min(v):8.2f}  max {max(v):8.2f}", flush=True)
