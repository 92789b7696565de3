"""One warm multiply of a BASELINE config through the C ABI (for ncu launch lists / captures).

python tools/dev/prof_run.py c4a [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np
import torch

import paper_1708_09746_b200 as G
from gf2x_synth import CONFIGS, batch_pair, operand_pair

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
bits, batch = CONFIGS[cfg]
if batch == 1:
    a, b = operand_pair(bits)
else:
    a, b = batch_pair(bits, batch)
da = torch.from_numpy(a.reshape(-1).view(np.int64)).cuda().view(torch.uint64)
db = torch.from_numpy(b.reshape(-1).view(np.int64)).cuda().view(torch.uint64)
for _ in range(reps):
    if batch == 1:
        G.gf2x_mul(da, bits, db, bits)
    else:
        G.gf2x_mul_batched(da, bits, db, bits, batch)
torch.cuda.synchronize()
print("launches per multiply:", G.gf2x_launch_count(bits, bits, batch))
