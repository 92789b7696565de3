"""Ad-hoc: device time of the sharded decomposition simulated on one GPU (all virtual ranks in sequence),
per-rank kernel breakdown via the profiling hook.  python tools/dev/gpu_shard_timing.py [bits]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_1708_09746_b200 as G
from gf2x_synth import operand_pair

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 29
a, b = operand_pair(bits)
da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
c = G.gf2x_mul(da, bits, db, bits)
for R in (2, 4, 8):
    for _ in range(2):
        G.gf2x_mul_sharded_sim(da, db, bits, R)
    torch.cuda.synchronize()
    G.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = G.gf2x_mul_sharded_sim(da, db, bits, R)
    e1.record()
    torch.cuda.synchronize()
    rep = G.profile_report()
    G.profile_enable(False)
    ok = torch.equal(out.view(torch.int64), c.view(torch.int64))
    print(f"G={R} sim total {e0.elapsed_time(e1):.3f} ms (all ranks in sequence) ok={ok}")
    for r in rep:
        print(f"    {r['kernel']:<22} {r['launches']:>3} launches {r['ms']:8.3f} ms  per rank {r['ms'] / R:7.3f}")
