"""Multi-process (world_size 2 and 4, gloo, CPU) tests of the sharded multiply's host-side logic.

The sharded multiply (include/gf2x.h gf2x_mul_sharded) moves data between
ranks by transfer lists every rank derives from (bits, G) (gf2x_shard_plan, host only).  Here real
processes execute those lists with gloo send/recv on element *labels* (global point indices) and check
the layouts they produce against the index maps the kernels use:
  blocked:   rank r holds points [r Nloc, (r+1) Nloc)
  pack:      element i of a blocked block -> chunk q = bits [K-g, K) of i, position
             j = (i & (2^(K-g)-1)) | ((i >> K) << (K-g))            (k_pack, shard.cuh)
  t-sliced:  rank q's local index li is global (li & (2^(K-g)-1)) | (q << (K-g)) | ((li >> (K-g)) << K)
             (IdxMap{K-g, g, q}, the multiplier index map of the top iFFT layers)
and that the cross-rank Taylor-step and halo lists pair up and stay inside the buffers; the peer-memory
all-to-all (k_pull_pack / k_pull_unpack: each rank reads every rank's buffer) is checked on the same labels.  Also the
128-byte NCCL-id broadcast helper over a gloo process group.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1708_09746_b200 as G


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _execute(plan_list, rank, bufs):
    """Run a transfer list on this rank: bufs maps buffer name -> int64 label array (16 B per element)."""
    reqs, recv_into = [], []
    for src, dst, sb, db, soff, doff, nbytes in plan_list:
        assert soff % 16 == 0 and doff % 16 == 0 and nbytes % 16 == 0 and nbytes > 0
        s0, d0, ne = soff // 16, doff // 16, nbytes // 16
        if src == rank and dst == rank:
            bufs[db][d0:d0 + ne] = bufs[sb][s0:s0 + ne].copy()
        elif src == rank:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(bufs[sb][s0:s0 + ne])), dst))
        elif dst == rank:
            t = torch.empty(ne, dtype=torch.int64)
            reqs.append(dist.irecv(t, src))
            recv_into.append((db, d0, ne, t))
    for r in reqs:
        r.wait()
    for db, d0, ne, t in recv_into:
        bufs[db][d0:d0 + ne] = t.numpy()


def _worker(rank, world, port, bits, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        plan = G.gf2x_shard_plan(bits, world)
        # every rank derives the same plan
        allp = [None] * world
        dist.all_gather_object(allp, json.dumps(plan, sort_keys=True))
        assert all(p == allp[0] for p in allp), "ranks derived different exchange plans"
        # the NCCL unique-id broadcast helper works over any process group
        uid = G.broadcast_unique_id(lambda: bytes(range(128)), rank)
        assert uid == bytes(range(128))

        # ---- forward: rank r gathers operand r & 1 (a: even ranks, b: odd) into A, converts it, and swaps
        # the converted operand with its partner r ^ 1 (into B)
        nb = {k: v // 16 for k, v in plan["buffers"].items()}
        n_units = plan["n"] // 2                       # 64-bit words, labelled per 16-byte unit
        sh = n_units // world
        lab_a = np.arange(n_units, dtype=np.int64)
        lab_b = lab_a + (1 << 40)
        bufs = {"IN_A": lab_a[rank * sh:(rank + 1) * sh].copy(), "IN_B": lab_b[rank * sh:(rank + 1) * sh].copy(),
                "A": np.full(nb["A"], -1, dtype=np.int64), "B": np.full(nb["B"], -1, dtype=np.int64)}
        _execute(plan["gather"], rank, bufs)
        assert np.array_equal(bufs["A"][:n_units], lab_b if rank & 1 else lab_a), "gathered operand"
        _execute(plan["xchg"], rank, bufs)
        assert np.array_equal(bufs["B"][:n_units], lab_a if rank & 1 else lab_b), "partner's operand"

        g, K, Nloc = plan["g"], plan["K"], plan["Nloc"]
        assert plan["G"] == world and (1 << g) == world
        Kg = K - g
        chunk = Nloc >> g
        idx = np.arange(Nloc, dtype=np.int64)
        # ---- blocked -> pack -> a2a_fwd -> t-sliced
        q_of = np.arange(world, dtype=np.int64)[:, None]
        j = np.arange(chunk, dtype=np.int64)[None, :]
        pack_src = (j & ((1 << Kg) - 1)) | (q_of << Kg) | ((j >> Kg) << K)          # [q, j] -> i
        X = np.full(nb["X"], -1, dtype=np.int64)
        X[:Nloc] = (rank * Nloc + pack_src).reshape(-1)
        T = np.full(nb["T"], -1, dtype=np.int64)
        bufs = {"X": X, "T": T}
        _execute(plan["a2a_fwd"], rank, bufs)
        want_t = (idx & ((1 << Kg) - 1)) | (rank << Kg) | ((idx >> Kg) << K)
        assert np.array_equal(bufs["T"][:Nloc], want_t), "t-sliced layout does not match IdxMap{K-g, g, q}"
        # ---- a2a_back -> unpack -> blocked
        bufs["X"][:] = -1
        _execute(plan["a2a_back"], rank, bufs)
        W = np.full(Nloc, -1, dtype=np.int64)
        W[pack_src.reshape(-1)] = bufs["X"][:Nloc]
        assert np.array_equal(W, rank * Nloc + idx), "blocked layout not restored"
        # ---- peer-memory path (k_pull_pack / k_pull_unpack): every rank reads the other ranks' buffers
        # (modelled by an all-gather of the buffers = what IPC mapping exposes), packing while it pulls
        Wb = torch.from_numpy(rank * Nloc + idx)
        allw = [torch.empty_like(Wb) for _ in range(world)]
        dist.all_gather(allw, Wb)
        Tp = np.concatenate([allw[r].numpy()[pack_src[rank]] for r in range(world)])   # T[r chunk + j]
        assert np.array_equal(Tp, want_t), "pull-pack: t-sliced layout"
        allt = [torch.empty_like(Wb) for _ in range(world)]
        dist.all_gather(allt, torch.from_numpy(Tp))
        Wp = np.full(Nloc, -1, dtype=np.int64)
        for q in range(world):
            Wp[pack_src[q]] = allt[q].numpy()[rank * chunk:(rank + 1) * chunk]
        assert np.array_equal(Wp, rank * Nloc + idx), "pull-unpack: blocked layout"
        # ---- cross-rank Taylor steps and halo: pairing and bounds
        lists = [("cross", c) for c in plan["cross"]] + [("halo", plan["halo"])]
        for name, lst in lists:
            for src, dst, sb, db, soff, doff, nbytes in lst:
                assert 0 <= src < world and 0 <= dst < world
                assert soff + nbytes <= plan["buffers"][sb] and doff + nbytes <= plan["buffers"][db], name
            # the halo carries the element just below the rank's first one (InterleavedCombine)
            bufs = {"W": np.full(nb["W"], -1, dtype=np.int64), "X": np.full(nb["X"], -1, dtype=np.int64),
                    "T": np.full(nb["T"], -1, dtype=np.int64), "HALO": np.full(nb["HALO"], -1, dtype=np.int64)}
            bufs["W"][:Nloc] = rank * Nloc + idx
            _execute(lst, rank, bufs)
            if name == "halo" and rank > 0:
                assert bufs["HALO"][0] == rank * Nloc - 1
        for li, l in enumerate(plan["top_cross"]):
            u = 1 << (l - 1 - K)
            h = 1 << (l - 1)
            d = h - u
            bufs = {"W": np.full(nb["W"], -1, dtype=np.int64), "X": np.full(nb["X"], -1, dtype=np.int64),
                    "T": np.full(nb["T"], -1, dtype=np.int64), "HALO": np.full(nb["HALO"], -1, dtype=np.int64)}
            bufs["W"][:Nloc] = rank * Nloc + idx
            _execute(plan["cross"][li], rank, bufs)
            gidx = rank * Nloc + idx
            pos = gidx % (2 * h)
            # phase B^-1 targets (position in [u, h)) read the element d above them (into X)
            tb = (pos >= u) & (pos < h)
            got = bufs["X"][:Nloc][tb]
            assert np.array_equal(got, gidx[tb] + d), f"level {l}: phase-B sources"
            # phase A^-1 targets (position in [h, h+u)) read the element d above them (into T)
            # (these targets start a block: h is a multiple of Nloc for levels above mloc)
            ta = (pos >= h) & (pos < h + u)
            if ta.any():
                assert idx[ta][0] == 0
                assert np.array_equal(bufs["T"][idx[ta]], gidx[ta] + d), f"level {l}: phase-A sources"
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        import traceback
        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,bits", [(2, 1 << 22), (2, 1 << 23), (4, 1 << 24)])
def test_exchange_plan_multiprocess(world, bits):
    G.load()
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bits, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_plan_rejects_unsupported_sizes():
    G.load()
    with pytest.raises(G.Gf2xError):
        G.gf2x_shard_plan(1 << 22, 3)        # G not a power of two
    with pytest.raises(G.Gf2xError):
        G.gf2x_shard_plan((1 << 22) + 64, 2)  # n not a power of two
    with pytest.raises(G.Gf2xError):
        G.gf2x_shard_plan(1 << 22, 8)        # too small for 8 ranks (m - g < K)
