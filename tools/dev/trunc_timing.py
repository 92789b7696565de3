"""Dev timing (not collected by pytest): the staircase with and without the truncated FFT.
python tools/dev/trunc_timing.py            (run twice: plain and with GF2X_NO_TRUNC=1)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import operand  # noqa: E402

for bits in [1 << 27, (1 << 27) + 64, (1 << 27) + (1 << 22), 1 << 28, (1 << 28) + 64, (1 << 28) + (1 << 23), 1 << 29]:
    a, b = operand(bits, seed=1), operand(bits, seed=2)
    da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
    c = G.gf2x_mul(da, bits, db, bits)
    for _ in range(3):
        G.gf2x_mul(da, bits, db, bits, c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        G.gf2x_mul(da, bits, db, bits, c)
    e1.record()
    torch.cuda.synchronize()
    print(f"{'no-trunc' if os.environ.get('GF2X_NO_TRUNC') else 'trunc'} bits={bits} ms={e0.elapsed_time(e1) / 10:.3f}", flush=True)
