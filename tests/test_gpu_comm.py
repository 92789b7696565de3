"""Failure surfacing of the multi-GPU communicator: ncclCommGetAsyncError is polled by
gf2x_comm_check / gf2x_comm_wait and before every sharded multiply; an aborted communicator makes every
later call fail with GF2X_ENCCL instead of hanging.  One GPU: a 1-rank NCCL communicator."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_09746_b200 as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1708_09746_b200 import build
    build.build()
    G.load()


def test_check_wait_abort():
    comm = G.Comm(G.Comm.unique_id(), 1, 0)
    try:
        comm.check()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            x = torch.ones(1 << 20, device="cuda")
            y = (x * 3).sum()
        comm.wait(s, timeout_s=60.0)          # idle-after-work stream: returns, no error
        assert float(y) == 3.0 * (1 << 20)
        comm.abort()
        with pytest.raises(G.Gf2xError, match="ENCCL"):
            comm.check()
        with pytest.raises(G.Gf2xError, match="ENCCL"):
            comm.wait(s, timeout_s=1.0)
        a = torch.zeros(1 << 10, dtype=torch.uint64, device="cuda")
        with pytest.raises(G.Gf2xError, match="ENCCL"):   # refused before anything is enqueued
            comm.mul(a, a, 1 << 16, torch.empty(2 << 10, dtype=torch.uint64, device="cuda"))
    finally:
        comm.close()
