"""Dev check (not collected by pytest): random large unequal sizes (2^20..2^27 bits) through gf2x_mul,
gf2x_mul_w(w=128) and gf2x_mul_alg4, checked on sampled output words (oracle single-word products) and modulo
random irreducible degree-64 polynomials."""
import random
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_1708_09746_b200 as G  # noqa: E402
from gf2x_synth import operand  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64).copy()).cuda().view(torch.uint64)


R = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
primes = O.random_irreducibles(2, seed=17)
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    ab = R.randrange(1 << 20, 1 << 27)
    bb = R.randrange(1 << 18, 1 << 27) if R.random() < 0.5 else ab
    a, b = operand(ab, seed=it * 7 + 1), operand(bb, seed=it * 7 + 2)
    for name, f in (("alg5", lambda: G.gf2x_mul(dev(a), ab, dev(b), bb)),
                    ("w128", lambda: G.gf2x_mul_w(dev(a), ab, dev(b), bb, w=128)),
                    ("alg4", lambda: G.gf2x_mul_alg4(dev(a), ab, dev(b), bb))):
        c = f()
        torch.cuda.synchronize()
        got = c.cpu().view(torch.int64).numpy().view(np.uint64).reshape(-1)
        n_out = len(got)
        ws = sorted({0, n_out - 1, n_out // 2} | {R.randrange(n_out) for _ in range(6)})
        ok = all(int(got[w]) == O.mul_word(a, b, w) for w in ws) and O.check_mod_p(a, b, got, primes)
        bad += not ok
        print(name, ab, bb, "ok" if ok else "MISMATCH", flush=True)
print("mismatches:", bad)
