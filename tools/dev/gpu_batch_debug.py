"""Ad-hoc: batched multiply vs oracle, listing mismatching pairs.  python tools/dev/gpu_batch_debug.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import oracle as O
import paper_1708_09746_b200 as G
from gf2x_synth import batch_pair


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


for bits, count in [(1 << 14, 4096), (1 << 14, 256), (1 << 14, 16), (1 << 12, 512), (1 << 16, 64)]:
    A, B = batch_pair(bits, count)
    want = np.stack([O.mul_karatsuba(A[i], B[i]) for i in range(count)])
    for rep in range(3):
        C = host(G.gf2x_mul_batched(dev(A), bits, dev(B), bits, count))
        bad = [i for i in range(count) if not np.array_equal(C[i], want[i])]
        print(bits, count, "rep", rep, "bad pairs", len(bad), bad[:20], flush=True)
        if bad:
            i = bad[0]
            w = np.nonzero(C[i] != want[i])[0]
            print("   pair", i, "bad words", w[:20], len(w), flush=True)
    # single multiplies of the first few bad pairs
    single_bad = 0
    for i in range(min(count, 300)):
        c = host(G.gf2x_mul(dev(A[i]), bits, dev(B[i]), bits))
        if not np.array_equal(c, want[i]):
            single_bad += 1
    print(bits, "single-call bad among first 300:", single_bad, flush=True)
