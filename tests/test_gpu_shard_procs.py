"""The partitioned multiply (gf2x_mul_sharded) executed by SEPARATE PROCESSES, one per rank,
on the one GPU this pool gives: a host-mode communicator (gf2x_comm_init_host) synchronises the ranks through
a gloo group, every exchange is a CUDA-IPC peer-memory pull kernel (k_pull_pack / k_pull_unpack and the peer
copies) over the other processes' mapped workspaces -- the real cross-process data path, with host barriers
in place of the NCCL ones (no kernel ever waits on another rank's kernel).  Each rank owns words
[r n/G, (r+1) n/G) of a and b and receives words [r 2n/G, (r+1) 2n/G) of c; the gathered product must equal
the oracle's (SHA-256 digest of the c3 product in tests/golden/oracle_digests.json)."""
import hashlib
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r'''
import os, sys, hashlib, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ".")
import paper_1708_09746_b200 as G
from gf2x_synth import CONFIGS, DEFAULT_SEED, operand_pair
torch.cuda.set_device(0)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
bits, _ = CONFIGS["c3"]
a, b = operand_pair(bits, DEFAULT_SEED)
lo, hi = G.shard_words(len(a), world, rank)
sa = torch.from_numpy(a[lo:hi].view(np.int64).copy()).cuda().view(torch.uint64)
sb = torch.from_numpy(b[lo:hi].view(np.int64).copy()).cuda().view(torch.uint64)
comm = G.Comm.from_host_group()
assert comm.peer_memory() in (0, 1)
for it in range(2):   # twice: the second call reuses the mapped workspaces
    sc = comm.mul(sa, sb, bits)
    torch.cuda.synchronize()
parts = [torch.empty(sc.numel(), dtype=torch.int64) for _ in range(world)]
dist.all_gather(parts, sc.cpu().view(torch.int64))
if rank == 0:
    c = torch.cat(parts).numpy().view(np.uint64)
    print("DIGEST", hashlib.sha256(c.astype("<u8").tobytes()).hexdigest(), comm.peer_memory(), flush=True)
dist.barrier()
comm.close()
dist.destroy_process_group()
'''


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_multiply_across_processes(world):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_digests.json")))["digests"]["c3"]["sha256"]
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", _CHILD], cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append((p.returncode, o, e))
    for rc, o, e in outs:
        assert rc == 0, e[-3000:]
    line = [l for l in outs[0][1].splitlines() if l.startswith("DIGEST")][0].split()
    assert line[1] == gold
    assert line[2] == "1"   # the exchanges ran as peer-memory pulls
