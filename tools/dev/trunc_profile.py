import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1708_09746_b200 as G
from gf2x_synth import operand
bits = (1 << 28) + 64
a, b = operand(bits, seed=1), operand(bits, seed=2)
da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64); db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
c = G.gf2x_mul(da, bits, db, bits)
for _ in range(3): G.gf2x_mul(da, bits, db, bits, c)
torch.cuda.synchronize()
G.profile_enable(True)
for _ in range(5): G.gf2x_mul(da, bits, db, bits, c)
for r in G.profile_report(): print(r['kernel'], r['launches'] // 5, round(r['ms'] / 5, 3))
