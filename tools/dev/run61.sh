#!/bin/bash
mkdir -p gpurun_out
L=paper_1708_09746_b200/libgf2x_b200.so
python tools/dev/ab_bench.py c4b 10 $L paper_1708_09746_b200/libgf2x_b200_rbs.so > gpurun_out/t61_c4b.txt 2>&1
GF2X_LIB=paper_1708_09746_b200/libgf2x_b200_rbs.so python -c "
import numpy as np, torch, sys
sys.path.insert(0,'.')
import paper_1708_09746_b200 as G, oracle as O
from gf2x_synth import operand_pair
G.load('paper_1708_09746_b200/libgf2x_b200_rbs.so')
for bits in (1<<20, 1<<23, (1<<22)+(1<<20)):
    a,b=operand_pair(bits)
    da=torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64); db=torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
    c=G.gf2x_mul(da,bits,db,bits); torch.cuda.synchronize()
    print(bits, np.array_equal(c.cpu().view(torch.int64).numpy().view(np.uint64), O.alg5_mul(a,bits,b,bits)))
" > gpurun_out/t61_parity.txt 2>&1
