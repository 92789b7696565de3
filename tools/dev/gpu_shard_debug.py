"""Ad-hoc: sharded-multiply simulation vs oracle.  python tools/dev/gpu_shard_debug.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import time

import numpy as np
import torch

import oracle as O
import paper_1708_09746_b200 as G
from gf2x_synth import operand_pair


def dev(x):
    return torch.from_numpy(x.view(np.int64).copy()).cuda().view(torch.uint64)


for bits, ranks in [(1 << 22, [2]), (1 << 23, [2, 4]), (1 << 24, [2, 4, 8])]:
    a, b = operand_pair(bits, seed=bits)
    want = O.mul_karatsuba(a, b)
    single = G.gf2x_mul(dev(a), bits, dev(b), bits).cpu().view(torch.int64).numpy().view(np.uint64)
    print(bits, "single ok", np.array_equal(single, want), flush=True)
    for R in ranks:
        try:
            c = G.gf2x_mul_sharded_sim(dev(a), dev(b), bits, R)
            torch.cuda.synchronize()
            got = c.cpu().view(torch.int64).numpy().view(np.uint64)
            bad = np.nonzero(got != want)[0]
            print(bits, R, "ok" if len(bad) == 0 else f"MISMATCH {len(bad)} first {bad[:8]} of {len(want)}", flush=True)
        except Exception as e:
            print(bits, R, "ERROR", e, flush=True)

# stage bisection
bits = 1 << 23
a, b = operand_pair(bits, seed=bits)
_, st = O.alg5_mul(a, bits, b, bits, stages=True)
for R in [2, 4]:
    for stage, key in [(1, "fft_a"), (5, "icvt")]:
        got = G.gf2x_debug_shard_stage(dev(a), dev(b), bits, R, stage).cpu().view(torch.int64).numpy().view(np.uint64).reshape(-1, 2)
        bad = np.nonzero(np.any(got != st[key], axis=1))[0]
        print("R", R, "stage", stage, "ok" if len(bad) == 0 else f"MISMATCH {len(bad)} first {bad[:6]} last {bad[-3:]}", flush=True)
