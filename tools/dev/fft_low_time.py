"""Time the warp-shuffle formulation of the five innermost forward FFT layers against k_bottom's bit-sliced
layers (2^24 points x 2 operands, c4b's size), CUDA events, median of 5 rounds of 10 launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_1708_09746_b200 as G
from gf2x_synth import splitmix64

m = 24
n = 1 << m
w = splitmix64(7, 4 * n).reshape(2, n, 2)
A = torch.from_numpy(w[0].view(np.int64).copy()).cuda().view(torch.uint64)
B = torch.from_numpy(w[1].view(np.int64).copy()).cuda().view(torch.uint64)
res = {0: [], 1: []}
for rnd in range(5):
    for v in (0, 1):
        for _ in range(2):
            G.experiment_fft_low(A, B, m, v)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            G.experiment_fft_low(A, B, m, v)
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1) / 10)
for v, name in ((0, "bit-sliced (k_bottom, L = 5, forward only)"), (1, "warp-shuffle (k_fft_low_shfl)")):
    print(f"{name:45s} median {np.median(res[v]):.4f} ms  min {min(res[v]):.4f}", flush=True)
