"""Small workload touching every kernel, for compute-sanitizer (racecheck / memcheck / synccheck).

python tools/dev/gpu_sanitize_run.py   -- checks the products against brute force / Karatsuba."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import oracle as O
import paper_1708_09746_b200 as G
from gf2x_synth import batch_pair, operand_pair


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


ok = True
for bits in (64 * 5 + 3, 1 << 12, 1 << 18, 1 << 22):
    a, b = operand_pair(bits, seed=bits)
    got = host(G.gf2x_mul(dev(a), bits, dev(b), bits))
    want = O.alg5_mul(a, bits, b, bits)
    ok &= bool(np.array_equal(got, want))
    print(bits, np.array_equal(got, want), flush=True)
A, B = batch_pair(1 << 14, 8)
C = host(G.gf2x_mul_batched(dev(A), 1 << 14, dev(B), 1 << 14, 8))
r = all(np.array_equal(C[i], O.mul_karatsuba(A[i], B[i])) for i in range(8))
ok &= r
print("batched", r, flush=True)
a, b = operand_pair(1 << 22, seed=3)
got = host(G.gf2x_mul_sharded_sim(dev(a), dev(b), 1 << 22, 2))
r = np.array_equal(got, O.mul_karatsuba(a, b))
ok &= bool(r)
print("sharded sim", r, flush=True)
print("ALL OK" if ok else "FAILURES")
sys.exit(0 if ok else 1)
