"""Dev timing (not collected by pytest): a long times a short operand, truncated vs full transform.
python tools/dev/trunc_unbalanced_timing.py   (and with GF2X_NO_TRUNC=1)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import operand  # noqa: E402

for ab, bb in [((1 << 28) + 64, 1 << 20), ((1 << 28) + 64, 1 << 26), ((1 << 27) + 64 * 3, 1 << 16)]:
    a, b = operand(ab, seed=1), operand(bb, seed=2)
    da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
    c = G.gf2x_mul(da, ab, db, bb)
    for _ in range(3):
        G.gf2x_mul(da, ab, db, bb, c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        G.gf2x_mul(da, ab, db, bb, c)
    e1.record()
    torch.cuda.synchronize()
    tag = "no-trunc" if os.environ.get("GF2X_NO_TRUNC") else "trunc"
    print(f"{tag} a={ab} b={bb} trunc_j={G.gf2x_plan(ab, bb)['trunc_j']} ms={e0.elapsed_time(e1) / 10:.3f}", flush=True)
