/*
 * gf2x.h -- C ABI of the B200 (sm_100a) GF(2)[x] multiplier (arXiv 1708.09746, Alg. 5).
 *
 * Operation (§2.1 P:211-214 and Alg. 5 input/output P:886-888): given binary polynomials
 * a(x), b(x) as bit sequences of lengths a_bits, b_bits, compute c(x) = a(x) * b(x) in GF(2)[x].
 * The product is computed by the paper's Alg. 5: Split into 64-bit blocks, BasisCvt
 * (Alg. 3) to the LCH novel polynomial basis, changeRepr into the tower field TGF(2^128) (§3.2),
 * FFT_LCH (Alg. 1) at 2^m points, pointwise products, iFFT_LCH, iBasisCvt, changeRepr back and
 * InterleavedCombine.  The result is exact and unique (no rounding).
 *
 * Packing (R12): little-endian 64-bit words; bit i of word j is the
 * coefficient of x^(64 j + i).  n_x = ceil(x_bits / 64) words per operand.  The product occupies
 * n_a + n_b words (R13); all of them are written, zero above degree a_bits+b_bits-2.
 * Bits of a/b at positions >= a_bits/b_bits are ignored.
 *
 * Memory: a, b, c (and ws) are DEVICE pointers owned by the caller.  c must not overlap a or b
 * (GF2X_EINVAL).  Calls are enqueued on `stream` and return after enqueue (no host sync in steady
 * state); kernel faults surface at the caller's next synchronisation.  The first call on a device
 * builds and uploads the constant tables (synchronous, once).
 *
 * Errors: every entry point returns a gf2x_status; detail text for the last error of the calling
 * thread is available from gf2x_last_error().  No C++ exception crosses this boundary.
 *
 * Size cap: FFT size N = 2^ceil(log2(n_a + n_b - 1)) <= 2^32 (multipliers stay in TGF(2^32),
 * §4.4); larger requests return GF2X_ETOOBIG.
 */
#ifndef GF2X_B200_H
#define GF2X_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GF2X_OK = 0,
    GF2X_EINVAL = 1,   /* bad argument: null pointer with nonzero size, aliasing, negative batch */
    GF2X_ETOOBIG = 2,  /* N > 2^32 or the workspace cannot be represented */
    GF2X_ENOMEM = 3,   /* device allocation failed / workspace too small */
    GF2X_ECUDA = 4,    /* CUDA runtime error (see gf2x_last_error) */
    GF2X_ENCCL = 5     /* NCCL error (multi-GPU entry points) */
} gf2x_status;

/* c = a * b.  `stream` is a cudaStream_t (0 = legacy default stream). */
gf2x_status gf2x_mul(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits,
                     uint64_t* c, void* stream);

/* `batch` independent products of equal sizes, operands contiguous:
 * a_i at a + i*n_a, b_i at b + i*n_b, c_i at c + i*(n_a+n_b).  batch == 0 is a no-op. */
gf2x_status gf2x_mul_batched(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits,
                             uint64_t* c, int64_t batch, void* stream);

/* Workspace bytes a call with these sizes needs (0 for empty products). */
size_t gf2x_workspace_bytes(uint64_t a_bits, uint64_t b_bits, int64_t batch);

/* As gf2x_mul_batched but with a caller-provided device workspace of ws_bytes
 * (>= gf2x_workspace_bytes, 256-byte aligned) instead of the library's per-stream cache. */
gf2x_status gf2x_mul_ws(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits,
                        uint64_t* c, int64_t batch, void* ws, size_t ws_bytes, void* stream);

/* Number of kernels one gf2x_mul_batched call with these sizes enqueues (for launch accounting). */
int gf2x_launch_count(uint64_t a_bits, uint64_t b_bits, int64_t batch);

/* Debug / parity hook: run only the forward pipeline up to a stage and copy the FFT-domain
 * intermediate of operand a into `out` (device, N*2 words, tower representation):
 *   stage 1 = after BasisCvt + changeRepr, 2 = after FFT_LCH, 3 = after pointmul,
 *   4 = after iFFT_LCH, 5 = after iBasisCvt (tower).  Returns EINVAL for other stages. */
gf2x_status gf2x_debug_stage(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits,
                             int stage, uint64_t* out, void* stream);

/* Block width (sec 4.2): Alg. 5 with w-bit blocks
 * over TGF(2^(2w)).  w = 64 is gf2x_mul_batched (TGF(2^128)); w = 128 splits the operands into
 * 128-bit blocks, converts them into TGF(2^256) = TGF(2^128)[x_8]/(x_8^2 + x_8 + v_127) through
 * GF(2)[z]/(z^256 + z^10 + z^5 + z^2 + 1) (R20) and runs the FFT on half as many points.
 * Same operands, output, memory and error contract as gf2x_mul_batched (the library's per-stream
 * workspace cache is used); EINVAL for other w.  The result is the same exact product. */
gf2x_status gf2x_mul_w(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                       int64_t batch, int w, void* stream);
/* kernels one gf2x_mul_w call enqueues (0 for unsupported w) */
int gf2x_launch_count_w(uint64_t a_bits, uint64_t b_bits, int64_t batch, int w);
/* w = 128 debug / parity hook: operand a's TGF(2^256) spectrum (N x 4 words, DEVICE; element i =
 * words 4i..4i+3, coordinates of v_0..v_255) after stage 1 (changeRepr), 2 (FFT_LCH), 3 (pointmul)
 * or 5 (iBasisCvt); N = 2^ceil(log2(ceil(a_bits/128) + ceil(b_bits/128) - 1)).  EINVAL otherwise. */
gf2x_status gf2x_debug_stage_w128(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, int stage,
                                  uint64_t* out, void* stream);

/* Alg. 4 (sec 3.1): the "simple" multiplication that keeps the
 * working field GF(2^128) in polynomial basis (no changeRepr) and runs FFT_LCH with the dense multipliers
 * psi^-1(s_k(phi_v(b))).  The same exact product as gf2x_mul_batched (same operands, output, memory and
 * error contract); it exists as the comparison point for the tower representation and is slower.
 * gf2x_debug_stage_alg4: operand a's spectrum (N x 2 words, polynomial basis, DEVICE) after stage 2
 * (FFT_LCH) or 3 (pointmul); EINVAL for other stages. */
gf2x_status gf2x_mul_alg4(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                          int64_t batch, void* stream);
gf2x_status gf2x_debug_stage_alg4(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, int stage,
                                  uint64_t* out, void* stream);

/* App. C, its first step: BasisCvt (Alg. 3 P:518-539 with Alg. 2
 * P:492-511; inverse if `inverse` != 0) on 2^M GF(2) coefficients, "proceeded straightforwardly with alg. 3"
 * (P:1523).  words: DEVICE, caller-owned, 2^(M-6) words, coefficient t = bit t % 64 of word t / 64 (the
 * packing of gf2x_mul's operands), converted in place; on return (stream-ordered) word bits are the
 * novel-basis coefficients g_t with f(x) = sum_t g_t X_t(x).  6 <= M <= 40, else GF2X_EINVAL. */
gf2x_status gf2x_basis_cvt_bits(uint64_t* words, int M, int inverse, void* stream);
/* App. C: c = a * b through the Frobenius bijection E_(beta_(m+64) + V_m), no Kronecker
 * segmentation: 2^m evaluation points with 128 * 2^m >= a_bits + b_bits - 1 (R23), FFT_LCH in the
 * polynomial basis with the displacement alpha = beta_(m+64).  Same operand / output packing and error
 * contract as gf2x_mul (a, b, c DEVICE; c receives ceil(a_bits/64) + ceil(b_bits/64) words; a zero-length
 * operand gives a zero product); its workspace is the per-stream one gf2x_mul keeps.  m <= 26, else
 * GF2X_ETOOBIG.  Exact; a comparison variant of the product path (slower on B200: DESIGN.md §10d). */
gf2x_status gf2x_mul_frob(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Multi-GPU: the FFT partitioned across G = nranks ranks, one process per GPU (the
 * decomposition is described in DESIGN.md §9).  NCCL is loaded at run time (libnccl.so.2).
 *
 * gf2x_comm_unique_id: on one rank, write the 128-byte NCCL unique id into id_out; the caller
 *   distributes it (e.g. torch.distributed broadcast) and every rank calls gf2x_comm_init with it
 *   on its own device (collective; blocks until all ranks joined).
 * gf2x_mul_sharded: a_bits = b_bits = bits, n = ceil(bits/64) must be a power of two and
 *   log2(2n) - log2(G) >= max(16, 12).  Rank r passes words [r n/G, (r+1) n/G) of a and b
 *   (DEVICE, caller-owned) and receives words [r 2n/G, (r+1) 2n/G) of c.  Enqueued on `stream`
 *   (collectives included); returns after enqueue, except that the first call for a size (which
 *   allocates the communicator's workspace and maps the peers' workspaces, see
 *   gf2x_comm_peer_memory) synchronises the stream.  EINVAL on unsupported sizes, ENCCL on NCCL
 *   errors.  The communicator owns a workspace, freed by gf2x_comm_destroy; G <= 8.
 * gf2x_mul_sharded_sim: the same algorithm with `nranks` virtual ranks in one process on the
 *   current device (data movement between ranks = device copies); a, b full operands, c the full
 *   2n-word product (DEVICE).  Used to check the decomposition bit-exactly on one GPU.
 * ------------------------------------------------------------------------------------------- */
typedef struct gf2x_comm_s* gf2x_comm_t;
gf2x_status gf2x_comm_unique_id(void* id_out);
gf2x_status gf2x_comm_init(const void* nccl_unique_id, int nranks, int rank, gf2x_comm_t* out);
gf2x_status gf2x_comm_destroy(gf2x_comm_t comm);
/* Exchange path of the communicator, fixed by its first gf2x_mul_sharded (and whenever the workspace
 * grows): 1 = peer memory (every rank's workspace mapped with CUDA IPC; the all-to-all is pulled and
 * (un)packed by one kernel over NVLink, the other exchanges are peer copies, ordering by stream-ordered
 * NCCL all-reduce barriers), 0 = NCCL grouped send/recv (IPC unavailable or GF2X_SHARD_NCCL=1; all ranks
 * agree), -1 = null comm. */
int gf2x_comm_peer_memory(gf2x_comm_t comm);
/* Failure surfacing.
 * gf2x_comm_check: GF2X_OK, or GF2X_ENCCL if NCCL reports an asynchronous error on the communicator
 *   (ncclCommGetAsyncError; e.g. a peer process died) -- the communicator is then aborted
 *   (ncclCommAbort, which also releases NCCL kernels blocked on the dead peer) and every later call
 *   on it returns GF2X_ENCCL.  gf2x_mul_sharded runs this check before it enqueues anything.
 * gf2x_comm_wait: host wait for `stream` that polls the stream and the asynchronous NCCL error every
 *   200 us; on an error, or after timeout_s seconds (<= 0: no timeout), the communicator is aborted
 *   and GF2X_ENCCL is returned instead of hanging in cudaStreamSynchronize.  GF2X_ECUDA on a
 *   stream fault.
 * gf2x_comm_abort: abort the communicator now (collective peers see an error, not a hang).  The
 *   handle must still be released with gf2x_comm_destroy. */
gf2x_status gf2x_comm_check(gf2x_comm_t comm);
/* Experiment (not on the product path): changeRepr^-1 of n tower elements P (16 bytes each, device)
 * into out (n x 16 bytes, device) as a tcgen05.mma kind::i8 product of 0/1 bytes with the accumulator in TMEM,
 * 128 elements per MMA tile.  lbo / sbo: the shared-memory descriptors' core-matrix offsets in bytes (0: the
 * canonical no-swizzle K-major values 128 / 1024).  Profiled as "k_ipsi_tc". */
gf2x_status gf2x_experiment_ipsi_tc(const void* P, uint64_t n, void* out, uint32_t lbo, uint32_t sbo, void* stream);

/* Measured experiment, not the product path: the five innermost forward FFT_LCH layers
 * (Alg. 1, layers k = 4 .. 0 of a 2^m-point transform, multipliers s_k(phi(b)) of the global block
 * bases), in place on two device arrays A, B of 2^m TGF(2^128) elements (uint4, tower representation),
 * 11 <= m <= 30.  variant 0: k_bottom's bit-sliced layers (the product path's formulation); variant 1: a
 * warp-shuffle formulation (one element per lane, partner lane ^ 2^k).  Both give the same result.
 * Stream-ordered; GF2X_EINVAL on bad arguments. */
gf2x_status gf2x_experiment_fft_low(void* A, void* B, uint32_t m, int variant, void* stream);

/* Host-mode communicator (no NCCL): the ranks' synchronisation goes through two caller-supplied HOST callbacks,
 * e.g. a torch.distributed gloo group.  `barrier(user)` returns when every rank has called it; `allgather(in,
 * out, bytes, user)` gathers `bytes` from every rank into out[rank * bytes].  Both return 0 on success.  All
 * exchanges of gf2x_mul_sharded are then peer-memory pulls of CUDA-IPC-mapped workspaces (GF2X_ECUDA when the
 * mapping fails, e.g. no peer access), each preceded by cudaStreamSynchronize + barrier; the ranks may share one
 * GPU (no kernel ever waits on another rank's kernel).  Meant for tests and hosts without NCCL; slower than the
 * stream-ordered NCCL barriers of gf2x_comm_init.  Callbacks are invoked from the calling thread only. */
typedef int (*gf2x_host_barrier_fn)(void* user);
typedef int (*gf2x_host_allgather_fn)(const void* in, void* out, size_t bytes, void* user);
gf2x_status gf2x_comm_init_host(int nranks, int rank, gf2x_host_barrier_fn barrier, gf2x_host_allgather_fn allgather,
                                void* user, gf2x_comm_t* out);
gf2x_status gf2x_comm_wait(gf2x_comm_t comm, void* stream, double timeout_s);
gf2x_status gf2x_comm_abort(gf2x_comm_t comm);
gf2x_status gf2x_mul_sharded(const uint64_t* a_shard, const uint64_t* b_shard, uint64_t bits,
                             uint64_t* c_shard, gf2x_comm_t comm, void* stream);
gf2x_status gf2x_mul_sharded_sim(const uint64_t* a, const uint64_t* b, uint64_t bits, uint64_t* c,
                                 int nranks, void* stream);
/* Debug / parity hook of the simulation: the concatenated rank blocks (N tower elements, N*2 words,
 * DEVICE) after stage 1 (forward FFT_LCH: evaluations in natural point order) or 5 (iBasisCvt). */
gf2x_status gf2x_debug_shard_stage(const uint64_t* a, const uint64_t* b, uint64_t bits, int nranks, int stage,
                                   uint64_t* out, void* stream);

/* Host-only description of the single-GPU plan (no device work): JSON into buf (cap bytes, NUL-terminated)
 * with m, N, the operand conversion sizes ma/mb, workspace bytes, the table FFT passes [c, k_lo, k_hi]
 * (forward order), the bit-sliced bottom layers, trunc_j (the truncated-FFT upper part is 2^trunc_j points, -1
 * if the product runs the full transform), and the BasisCvt / iBasisCvt passes (kind res / rb / tile /
 * stream, each with its Taylor steps [level, K] in forward execution order).  Returns the length needed, or
 * -1 for empty operands / unsupported sizes. */
int gf2x_plan(uint64_t a_bits, uint64_t b_bits, int64_t batch, char* buf, size_t cap);

/* Host-only description of the sharded multiply's exchanges (no device work): writes JSON into buf
 * (cap bytes, NUL-terminated) with the geometry (G, g, m, mloc, K, n, N, Nloc, per-rank buffer
 * sizes) and every transfer list [src_rank, dst_rank, src_buf, dst_buf, src_off, dst_off, bytes]
 * ("a2a_fwd", "a2a_back", "cross" per level of "top_cross", "halo") that every rank derives
 * identically.  Returns the length needed, or -1 if (bits, nranks) is unsupported. */
int gf2x_shard_plan(uint64_t bits, int nranks, char* buf, size_t cap);

/* Measurement hook (bench.py): while enabled, every kernel the library enqueues from the calling
 * thread is bracketed by CUDA events on its stream.  gf2x_profile_report synchronises those events
 * and writes a JSON array into buf (cap bytes, NUL-terminated):
 *   [{"kernel": name, "launches": n, "ms": total device ms, "bytes": algorithmic HBM bytes,
 *     "alu_ops": algorithmic ALU-pipe lane instructions (0 for kernels designed to be HBM-bound)}, ...]
 * and returns the length needed (call again with a larger buf if it exceeds cap).  Enabling or
 * disabling clears the record. */
gf2x_status gf2x_profile_enable(int on);
int gf2x_profile_report(char* buf, size_t cap);

const char* gf2x_status_string(gf2x_status s);
const char* gf2x_last_error(void);      /* thread-local detail text of the last failure */
gf2x_status gf2x_release(int device);   /* free cached workspaces and constant tables of a device */
const char* gf2x_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GF2X_B200_H */
