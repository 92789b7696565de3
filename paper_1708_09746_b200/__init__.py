"""B200-native GF(2)[x] multiplication (arXiv 1708.09746, Alg. 5) -- thin Python binding.

The binding only marshals arguments into the C ABI of include/gf2x.h (libgf2x_b200.so, built
in-tree for sm_100a by build.py).  Every step of the multiplication runs in the library's CUDA
kernels; there is no CPU fallback: if the shared library is missing or fails to load, importing
the compute entry points raises.

Tensors are torch.uint64 (or int64 reinterpreted) CUDA tensors holding little-endian 64-bit words,
bit i of word j = coefficient of x^(64 j + i).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgf2x_b200.so")

STATUS = {0: "GF2X_OK", 1: "GF2X_EINVAL", 2: "GF2X_ETOOBIG", 3: "GF2X_ENOMEM", 4: "GF2X_ECUDA", 5: "GF2X_ENCCL"}

# every symbol include/gf2x.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "gf2x_mul", "gf2x_mul_batched", "gf2x_workspace_bytes", "gf2x_mul_ws", "gf2x_launch_count",
    "gf2x_debug_stage", "gf2x_comm_unique_id", "gf2x_comm_init", "gf2x_comm_destroy", "gf2x_mul_sharded",
    "gf2x_mul_sharded_sim", "gf2x_debug_shard_stage", "gf2x_shard_plan", "gf2x_profile_enable", "gf2x_profile_report", "gf2x_status_string", "gf2x_last_error",
    "gf2x_release", "gf2x_version", "gf2x_mul_w", "gf2x_launch_count_w", "gf2x_debug_stage_w128",
    "gf2x_comm_peer_memory", "gf2x_mul_alg4", "gf2x_debug_stage_alg4", "gf2x_plan", "gf2x_basis_cvt_bits",
    "gf2x_mul_frob", "gf2x_comm_check", "gf2x_comm_wait", "gf2x_comm_abort", "gf2x_comm_init_host",
    "gf2x_experiment_ipsi_tc",
    "gf2x_experiment_fft_low",
]


class Gf2xError(RuntimeError):
    pass


_lib = None


def load(path: str = LIB_PATH):
    """Load libgf2x_b200.so (raises if it is absent: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise Gf2xError(f"{path} not built; run python -m paper_1708_09746_b200.build")
    L = ctypes.CDLL(path)
    u64, i64, vp, i32, sz = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.gf2x_mul.argtypes = [vp, u64, vp, u64, vp, vp]
    L.gf2x_mul_batched.argtypes = [vp, u64, vp, u64, vp, i64, vp]
    L.gf2x_workspace_bytes.argtypes = [u64, u64, i64]
    L.gf2x_workspace_bytes.restype = sz
    L.gf2x_mul_ws.argtypes = [vp, u64, vp, u64, vp, i64, vp, sz, vp]
    L.gf2x_launch_count.argtypes = [u64, u64, i64]
    L.gf2x_debug_stage.argtypes = [vp, u64, vp, u64, i32, vp, vp]
    L.gf2x_mul_w.argtypes = [vp, u64, vp, u64, vp, i64, i32, vp]
    L.gf2x_mul_w.restype = i32
    L.gf2x_launch_count_w.argtypes = [u64, u64, i64, i32]
    L.gf2x_debug_stage_w128.argtypes = [vp, u64, vp, u64, i32, vp, vp]
    L.gf2x_debug_stage_w128.restype = i32
    L.gf2x_mul_alg4.argtypes = [vp, u64, vp, u64, vp, i64, vp]
    L.gf2x_mul_alg4.restype = i32
    L.gf2x_basis_cvt_bits.argtypes = [vp, i32, i32, vp]
    L.gf2x_basis_cvt_bits.restype = i32
    L.gf2x_mul_frob.argtypes = [vp, u64, vp, u64, vp, vp]
    L.gf2x_mul_frob.restype = i32
    L.gf2x_debug_stage_alg4.argtypes = [vp, u64, vp, u64, i32, vp, vp]
    L.gf2x_debug_stage_alg4.restype = i32
    L.gf2x_status_string.argtypes = [i32]
    L.gf2x_status_string.restype = ctypes.c_char_p
    L.gf2x_last_error.restype = ctypes.c_char_p
    L.gf2x_release.argtypes = [i32]
    L.gf2x_version.restype = ctypes.c_char_p
    L.gf2x_comm_unique_id.argtypes = [vp]
    L.gf2x_comm_init.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    L.gf2x_comm_destroy.argtypes = [vp]
    L.gf2x_comm_peer_memory.argtypes = [vp]
    if hasattr(L, "gf2x_experiment_fft_low"):
        L.gf2x_experiment_fft_low.argtypes = [vp, vp, ctypes.c_uint32, i32, vp]
        L.gf2x_experiment_fft_low.restype = i32
    if hasattr(L, "gf2x_experiment_ipsi_tc"):
        L.gf2x_experiment_ipsi_tc.argtypes = [vp, u64, vp, ctypes.c_uint32, ctypes.c_uint32, vp]
        L.gf2x_experiment_ipsi_tc.restype = i32
    if hasattr(L, "gf2x_comm_init_host"):
        L.gf2x_comm_init_host.argtypes = [i32, i32, vp, vp, vp, ctypes.POINTER(vp)]
        L.gf2x_comm_init_host.restype = i32
    if hasattr(L, "gf2x_comm_check"):   # (older builds, loaded by the A/B tools, lack these)
        L.gf2x_comm_check.argtypes = [vp]
        L.gf2x_comm_wait.argtypes = [vp, vp, ctypes.c_double]
        L.gf2x_comm_abort.argtypes = [vp]
    L.gf2x_mul_sharded.argtypes = [vp, vp, u64, vp, vp, vp]
    L.gf2x_mul_sharded_sim.argtypes = [vp, vp, u64, vp, i32, vp]
    L.gf2x_debug_shard_stage.argtypes = [vp, vp, u64, i32, i32, vp, vp]
    for name in ("gf2x_comm_unique_id", "gf2x_comm_init", "gf2x_comm_destroy", "gf2x_mul_sharded", "gf2x_mul_sharded_sim",
                 "gf2x_debug_shard_stage", "gf2x_comm_check", "gf2x_comm_wait", "gf2x_comm_abort"):
        if hasattr(L, name):
            getattr(L, name).restype = i32
    L.gf2x_plan.argtypes = [u64, u64, i64, ctypes.c_char_p, sz]
    L.gf2x_plan.restype = i32
    L.gf2x_shard_plan.argtypes = [u64, i32, ctypes.c_char_p, sz]
    L.gf2x_shard_plan.restype = i32
    L.gf2x_profile_enable.argtypes = [i32]
    L.gf2x_profile_enable.restype = i32
    L.gf2x_profile_report.argtypes = [ctypes.c_char_p, sz]
    L.gf2x_profile_report.restype = i32
    for name in ("gf2x_mul", "gf2x_mul_batched", "gf2x_mul_ws", "gf2x_debug_stage", "gf2x_release"):
        getattr(L, name).restype = i32
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        detail = load().gf2x_last_error().decode()
        raise Gf2xError(f"{STATUS.get(status, status)}: {detail}")


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    if t is None:
        return None
    import torch
    assert t.is_cuda and t.is_contiguous() and t.dtype in (torch.uint64, torch.int64), "need contiguous CUDA 64-bit words"
    return ctypes.c_void_p(t.data_ptr())


def nwords(bits: int) -> int:
    return (bits + 63) // 64


def gf2x_mul(a, a_bits: int, b, b_bits: int, c=None, stream=None):
    """c = a * b over GF(2); a, b CUDA word tensors; returns c (n_a + n_b words)."""
    import torch
    if c is None:
        c = torch.empty(nwords(a_bits) + nwords(b_bits), dtype=torch.uint64, device=a.device)
    _check(load().gf2x_mul(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), _stream_ptr(stream)))
    return c


def gf2x_mul_batched(a, a_bits: int, b, b_bits: int, batch: int, c=None, stream=None):
    """`batch` products; a is (batch, n_a) (or flat), b (batch, n_b); returns (batch, n_a + n_b)."""
    import torch
    n_out = nwords(a_bits) + nwords(b_bits)
    if c is None:
        c = torch.empty(batch, n_out, dtype=torch.uint64, device=a.device)
    _check(load().gf2x_mul_batched(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), batch, _stream_ptr(stream)))
    return c


def gf2x_mul_w(a, a_bits: int, b, b_bits: int, w: int = 128, batch: int = 1, c=None, stream=None):
    """Alg. 5 with w-bit blocks (w = 64: TGF(2^128); w = 128: TGF(2^256)); same layout as gf2x_mul_batched."""
    import torch
    n_out = nwords(a_bits) + nwords(b_bits)
    if c is None:
        c = torch.empty(batch, n_out, dtype=torch.uint64, device=a.device)
    _check(load().gf2x_mul_w(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), batch, w, _stream_ptr(stream)))
    return c


def gf2x_launch_count_w(a_bits: int, b_bits: int, batch: int = 1, w: int = 128) -> int:
    return int(load().gf2x_launch_count_w(a_bits, b_bits, batch, w))


def gf2x_debug_stage_w128(a, a_bits: int, b, b_bits: int, stage: int, stream=None):
    """w = 128: operand a's TGF(2^256) spectrum (N, 4) after `stage` (1, 2, 3 or 5)."""
    import torch
    L = (a_bits + 127) // 128 + (b_bits + 127) // 128 - 1
    N = 1 << max(0, (L - 1).bit_length())
    out = torch.empty(N, 4, dtype=torch.uint64, device=a.device)
    _check(load().gf2x_debug_stage_w128(_ptr(a), a_bits, _ptr(b), b_bits, stage, _ptr(out), _stream_ptr(stream)))
    return out


def gf2x_mul_frob(a, a_bits: int, b, b_bits: int, c=None, stream=None):
    """App. C: c = a * b through the Frobenius bijection (same packing as gf2x_mul); returns c."""
    import torch
    if c is None:
        c = torch.empty(nwords(a_bits) + nwords(b_bits), dtype=torch.uint64, device=a.device)
    _check(load().gf2x_mul_frob(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), _stream_ptr(stream)))
    return c


def gf2x_basis_cvt_bits(words, M: int, inverse: bool = False, stream=None):
    """App. C's BasisCvt on 2^M GF(2) coefficients packed in a CUDA word tensor (2^(M-6) words), in place."""
    _check(load().gf2x_basis_cvt_bits(_ptr(words), M, 1 if inverse else 0, _stream_ptr(stream)))
    return words


def gf2x_mul_alg4(a, a_bits: int, b, b_bits: int, batch: int = 1, c=None, stream=None):
    """Alg. 4 (GF(2^128) polynomial basis, dense multipliers): the comparison variant; same layout."""
    import torch
    n_out = nwords(a_bits) + nwords(b_bits)
    if c is None:
        c = torch.empty(batch, n_out, dtype=torch.uint64, device=a.device)
    _check(load().gf2x_mul_alg4(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), batch, _stream_ptr(stream)))
    return c


def gf2x_debug_stage_alg4(a, a_bits: int, b, b_bits: int, stage: int, stream=None):
    import torch
    L = nwords(a_bits) + nwords(b_bits) - 1
    N = 1 << max(0, (L - 1).bit_length())
    out = torch.empty(N, 2, dtype=torch.uint64, device=a.device)
    _check(load().gf2x_debug_stage_alg4(_ptr(a), a_bits, _ptr(b), b_bits, stage, _ptr(out), _stream_ptr(stream)))
    return out


def gf2x_workspace_bytes(a_bits: int, b_bits: int, batch: int = 1) -> int:
    return int(load().gf2x_workspace_bytes(a_bits, b_bits, batch))


def gf2x_mul_ws(a, a_bits: int, b, b_bits: int, c, batch: int, ws, stream=None):
    _check(load().gf2x_mul_ws(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), batch,
                              ctypes.c_void_p(ws.data_ptr()), ws.numel() * ws.element_size(), _stream_ptr(stream)))
    return c


def gf2x_launch_count(a_bits: int, b_bits: int, batch: int = 1) -> int:
    return int(load().gf2x_launch_count(a_bits, b_bits, batch))


def gf2x_debug_stage(a, a_bits: int, b, b_bits: int, stage: int, stream=None):
    """FFT-domain intermediate of operand a (tower representation) after `stage` (1..5)."""
    import torch
    L = (nwords(a_bits) + nwords(b_bits) - 1)
    N = 1 << max(0, (L - 1).bit_length())
    out = torch.empty(N, 2, dtype=torch.uint64, device=a.device)
    _check(load().gf2x_debug_stage(_ptr(a), a_bits, _ptr(b), b_bits, stage, _ptr(out), _stream_ptr(stream)))
    return out


def gf2x_mul_sharded_sim(a, b, bits: int, nranks: int, c=None, stream=None):
    """The multi-GPU algorithm with `nranks` virtual ranks on this device (full a, b in; full c out)."""
    import torch
    if c is None:
        c = torch.empty(2 * nwords(bits), dtype=torch.uint64, device=a.device)
    _check(load().gf2x_mul_sharded_sim(_ptr(a), _ptr(b), bits, _ptr(c), nranks, _stream_ptr(stream)))
    return c


def gf2x_debug_shard_stage(a, b, bits: int, nranks: int, stage: int, stream=None):
    import torch
    N = 2 * nwords(bits)
    out = torch.empty(N, 2, dtype=torch.uint64, device=a.device)
    _check(load().gf2x_debug_shard_stage(_ptr(a), _ptr(b), bits, nranks, stage, _ptr(out), _stream_ptr(stream)))
    return out


def experiment_ipsi_tc(P, lbo: int = 0, sbo: int = 0, stream=None):
    """changeRepr^-1 of the tower elements P ((n, 2) uint64 / 16 bytes each, device) on the tensor cores
    (tcgen05.mma kind::i8, TMEM accumulator): the DESIGN.md §7 experiment.  Returns (n, 2) uint64."""
    import torch
    out = torch.empty_like(P)
    _check(load().gf2x_experiment_ipsi_tc(_ptr(P), P.shape[0], _ptr(out), lbo, sbo, _stream_ptr(stream)))
    return out


class Comm:
    """NCCL communicator of the library (one rank per process/GPU).

    The 128-byte unique id is created by rank 0 (`unique_id()`) and must reach every rank before
    `Comm(uid, nranks, rank)`; `init_from_process_group` does that with a torch.distributed broadcast.
    """

    def __init__(self, uid: bytes, nranks: int, rank: int):
        assert len(uid) == 128
        self.nranks, self.rank = nranks, rank
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, 128)
        _check(load().gf2x_comm_init(buf, nranks, rank, ctypes.byref(h)))
        self.handle = h

    @classmethod
    def from_host_group(cls, group=None):
        """Host-mode communicator (gf2x_comm_init_host): barriers and the IPC-handle exchange through a
        torch.distributed group (e.g. gloo), exchanges as peer-memory pulls; the ranks may share a GPU."""
        import torch
        import torch.distributed as dist
        self = cls.__new__(cls)
        self.nranks, self.rank = dist.get_world_size(group), dist.get_rank(group)
        BAR = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)
        AG = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)

        def _barrier(_user):
            try:
                dist.barrier(group=group)
                return 0
            except Exception:
                return 1

        def _allgather(src, dst, nbytes, _user):
            try:
                t = torch.frombuffer(bytearray(ctypes.string_at(src, nbytes)), dtype=torch.uint8)
                outs = [torch.empty_like(t) for _ in range(self.nranks)]
                dist.all_gather(outs, t, group=group)
                buf = b"".join(bytes(o.tolist()) for o in outs)
                ctypes.memmove(dst, buf, len(buf))
                return 0
            except Exception:
                return 1

        self._cbs = (BAR(_barrier), AG(_allgather))   # kept alive as long as the communicator
        h = ctypes.c_void_p()
        _check(load().gf2x_comm_init_host(self.nranks, self.rank, ctypes.cast(self._cbs[0], ctypes.c_void_p),
                                          ctypes.cast(self._cbs[1], ctypes.c_void_p), None, ctypes.byref(h)))
        self.handle = h
        return self

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load().gf2x_comm_unique_id(buf))
        return buf.raw

    def mul(self, a_shard, b_shard, bits: int, c_shard=None, stream=None):
        """Sharded product: this rank's words of a and b in, its 2n/G words of c out."""
        import torch
        if c_shard is None:
            c_shard = torch.empty(2 * nwords(bits) // self.nranks, dtype=torch.uint64, device=a_shard.device)
        _check(load().gf2x_mul_sharded(_ptr(a_shard), _ptr(b_shard), bits, _ptr(c_shard), self.handle,
                                       _stream_ptr(stream)))
        return c_shard

    def peer_memory(self) -> int:
        """1: exchanges over peer memory (CUDA IPC / NVLink), 0: NCCL send/recv (see include/gf2x.h)."""
        return int(load().gf2x_comm_peer_memory(self.handle))

    def check(self):
        """Raise if NCCL reports an asynchronous error (the communicator is then aborted)."""
        _check(load().gf2x_comm_check(self.handle))

    def wait(self, stream=None, timeout_s: float = 0.0):
        """Wait for `stream` while watching for asynchronous NCCL errors; abort + raise on error or timeout."""
        _check(load().gf2x_comm_wait(self.handle, _stream_ptr(stream), float(timeout_s)))

    def abort(self):
        _check(load().gf2x_comm_abort(self.handle))

    def close(self):
        if self.handle:
            _check(load().gf2x_comm_destroy(self.handle))
            self.handle = None


def broadcast_unique_id(uid_fn, rank: int, group=None) -> bytes:
    """Rank 0 calls uid_fn() (128 bytes); every rank returns the same bytes via torch.distributed."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t[:] = torch.frombuffer(bytearray(uid_fn()), dtype=torch.uint8)
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


def init_from_process_group(group=None) -> Comm:
    import torch.distributed as dist
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    uid = broadcast_unique_id(Comm.unique_id, rank, group)
    return Comm(uid, nranks, rank)


def shard_words(total_words: int, nranks: int, rank: int):
    """[lo, hi) word range of rank `rank` for an operand of total_words (block distribution)."""
    assert total_words % nranks == 0
    per = total_words // nranks
    return rank * per, (rank + 1) * per


def gf2x_plan(a_bits: int, b_bits: int, batch: int = 1) -> dict:
    """Host-only: the single-GPU plan (FFT passes, bottom layers, conversion passes; see include/gf2x.h)."""
    import json
    L = load()
    need = L.gf2x_plan(a_bits, b_bits, batch, None, 0)
    if need < 0:
        raise Gf2xError(f"GF2X_EINVAL: no plan for ({a_bits}, {b_bits}, {batch})")
    buf = ctypes.create_string_buffer(need + 16)
    L.gf2x_plan(a_bits, b_bits, batch, buf, len(buf))
    return json.loads(buf.value.decode())


def gf2x_shard_plan(bits: int, nranks: int) -> dict:
    """Host-only: geometry and exchange lists of the sharded multiply (see include/gf2x.h)."""
    import json
    L = load()
    need = L.gf2x_shard_plan(bits, nranks, None, 0)
    if need < 0:
        raise Gf2xError(f"GF2X_EINVAL: unsupported sharded size (bits={bits}, nranks={nranks})")
    buf = ctypes.create_string_buffer(need + 16)
    L.gf2x_shard_plan(bits, nranks, buf, len(buf))
    return json.loads(buf.value.decode())


def gf2x_release(device: int = 0):
    _check(load().gf2x_release(device))


def profile_enable(on: bool = True):
    _check(load().gf2x_profile_enable(1 if on else 0))


def profile_report():
    """Per-kernel device time (CUDA events) recorded since profile_enable(True)."""
    import json
    L = load()
    need = L.gf2x_profile_report(None, 0)
    buf = ctypes.create_string_buffer(need + 16)
    L.gf2x_profile_report(buf, len(buf))
    return json.loads(buf.value.decode())


def version() -> str:
    return load().gf2x_version().decode()


def experiment_fft_low(A, B, m: int, variant: int, stream=None):
    """The five innermost forward FFT layers of a 2^m-point transform, in place on A and B ((2^m, 2) uint64
    device tensors, tower elements): variant 0 bit-sliced (k_bottom), 1 warp-shuffle (DESIGN.md §7 experiment)."""
    _check(load().gf2x_experiment_fft_low(_ptr(A), _ptr(B), m, variant, _stream_ptr(stream)))
