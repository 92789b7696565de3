"""Phase timeline of k_small (SM_TRACE variant build): python tools/dev/small_trace.py [bits] [CL]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from paper_1708_09746_b200 import build
path = os.path.join(os.path.dirname(build.LIB), "libgf2x_b200_trace.so")
if not os.path.exists(path):
    path = build.build_variant("trace", ["SM_TRACE"])
import paper_1708_09746_b200 as G
G.load(path)
from gf2x_synth import operand_pair

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
os.environ["GF2X_SMALL_CL"] = sys.argv[2] if len(sys.argv) > 2 else "16"
a, b = operand_pair(bits)
da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
names = ["start", "tables+consts", "split", "BasisCvt", "psi", "fwd cross", "local FFT + sync", "transpose",
         "products", "combine + sync", "local iFFT", "inv cross + low^-1 + sync", "gather", "iBasisCvt + sync",
         "ipsi", "final sync"]
lib = ctypes.CDLL(path)
acc = []
for it in range(20):
    G.gf2x_mul(da, bits, db, bits)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 256)()
    assert lib.gf2x_debug_small_trace(buf) == 0
    t = np.array(buf[:], dtype=np.float64).reshape(16, 16)
    if it >= 5:
        acc.append(t)
t = np.median(np.array(acc), axis=0)
ncta = int(os.environ["GF2X_SMALL_CL"])
t0 = t[:ncta, 0].min()
print(f"bits {bits} CL {ncta}: per phase, us since the first CTA start (min / max over CTAs), median of 15 launches")
prev = None
for i, n in enumerate(names):
    col = t[:ncta, i] - t0
    if np.all(t[:ncta, i] == 0):
        continue
    print(f"{i:2d} {n:28s} {col.min() / 1000:7.2f} {col.max() / 1000:7.2f}")
