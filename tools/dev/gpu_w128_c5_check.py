import numpy as np, torch, time, sys
sys.path.insert(0, '.')
import oracle as O, paper_1708_09746_b200 as G
from gf2x_synth import CONFIGS, operand_pair
bits,_=CONFIGS['c5']
a,b=operand_pair(bits)
da=torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64); db=torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
c=G.gf2x_mul_w(da,bits,db,bits,w=128); torch.cuda.synchronize()
t=time.time(); c=G.gf2x_mul_w(da,bits,db,bits,w=128); torch.cuda.synchronize(); print('w128 c5 ms', (time.time()-t)*1e3)
got=c.cpu().view(torch.int64).numpy().view(np.uint64).reshape(-1)
n=len(a); rng=np.random.default_rng(3)
for w in sorted({0,n-1,n,2*n-1}|set(int(x) for x in rng.integers(0,2*n,size=4))):
    assert int(got[w])==O.mul_word(a,b,w), w
print('sampled ok; mod p', O.check_mod_p(a,b,got,O.random_irreducibles(2,seed=7)))
