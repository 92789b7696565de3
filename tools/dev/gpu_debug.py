"""Ad-hoc GPU debugging aid: stage-by-stage comparison of the CUDA path with the oracle.

python tools/dev/gpu_debug.py [bits ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import time

import numpy as np
import torch

import oracle as O
import paper_1708_09746_b200 as G
from gf2x_synth import operand_pair


def to_dev(x):
    return torch.from_numpy(x.view(np.int64).copy()).cuda().view(torch.uint64)


def to_np(t):
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def check(bits, stages=True):
    a, b = operand_pair(bits, seed=bits)
    da, db = to_dev(a), to_dev(b)
    c = to_np(G.gf2x_mul(da, bits, db, bits))
    torch.cuda.synchronize()
    want, st = O.alg5_mul(a, bits, b, bits, stages=True)
    ok = np.array_equal(c, want)
    print(f"bits={bits} product_ok={ok}", flush=True)
    if not ok and stages:
        names = {1: "cvt_a", 2: "fft_a", 3: "prod", 4: "ifft", 5: "icvt"}
        for s, nm in names.items():
            got = to_np(G.gf2x_debug_stage(da, bits, db, bits, s))
            torch.cuda.synchronize()
            eq = np.array_equal(got.reshape(-1, 2), st[nm])
            bad = np.nonzero(np.any(got.reshape(-1, 2) != st[nm], axis=1))[0]
            print(f"   stage {s} {nm}: {'ok' if eq else 'MISMATCH'} first bad {bad[:8]} of {len(bad)}", flush=True)
            if not eq:
                break
        bad = np.nonzero(c != want)[0]
        print("   product first bad words", bad[:10], "of", len(bad))
    return ok


if __name__ == "__main__":
    sizes = [int(x) for x in sys.argv[1:]] or [1, 64, 65, 128, 200, 1000, 4096, 1 << 12, 1 << 14, 1 << 16, 1 << 17, 1 << 20]
    t = time.time()
    allok = all([check(s) for s in sizes])
    print("ALL OK" if allok else "FAILURES", f"{time.time() - t:.1f}s")
