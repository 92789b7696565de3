"""Time the tensor-core changeRepr^-1 experiment against the product's bit-sliced k_ipsi_bs on 2^24 elements
(c4b's spectrum), CUDA events; also tries the swapped descriptor offsets if the default does not validate."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import oracle as O
import paper_1708_09746_b200 as G
from gf2x_synth import CONFIGS, operand_pair, splitmix64

n = 1 << 24
w = splitmix64(99, 2 * n).reshape(n, 2)
P = torch.from_numpy(w.view(np.int64).copy()).cuda().view(torch.uint64)
for lbo, sbo in [(0, 0)]:
    out = G.experiment_ipsi_tc(P, lbo, sbo)
    torch.cuda.synchronize()
    got = out[:64].cpu().view(torch.int64).numpy().view(np.uint64)
    ok = all((int(got[i, 0]) | (int(got[i, 1]) << 64)) == O.psi_inv(int(w[i, 0]) | (int(w[i, 1]) << 64)) for i in range(64))
    print("lbo/sbo", lbo, sbo, "correct" if ok else "WRONG", flush=True)
    if not ok:
        continue
    for _ in range(3):
        G.experiment_ipsi_tc(P, lbo, sbo)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        G.experiment_ipsi_tc(P, lbo, sbo)
    e1.record()
    torch.cuda.synchronize()
    print(f"tcgen05 kind::i8 psi^-1, 2^24 elements: {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)
# the product path's bit-sliced changeRepr^-1 + combine at c4b (profiled multiply)
bits, _ = CONFIGS["c4b"]
a, b = operand_pair(bits)
da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
for _ in range(2):
    G.gf2x_mul(da, bits, db, bits)
torch.cuda.synchronize()
G.profile_enable(True)
for _ in range(5):
    G.gf2x_mul(da, bits, db, bits)
torch.cuda.synchronize()
rep = {r["kernel"]: r["ms"] / r["launches"] for r in G.profile_report()}
G.profile_enable(False)
print(f"k_ipsi_bs (bit-sliced psi^-1 + combine), 2^24 elements: {rep['k_ipsi_bs']:.4f} ms", flush=True)
