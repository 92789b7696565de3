// shard.cuh -- the FFT partitioned across G ranks, included by gf2x.cu.
//
// G = 2^g ranks, operands of n = 2^p words (N = 2n points, m = p + 1), rank r owns the points
// [r N/G, (r+1) N/G) (index bits [m-g, m) = r, "blocked"), Nloc = N/G, mloc = m - g.
//
// Forward.  Every rank gathers both operands and converts them (BasisCvt, redundant).  With
// g(X) = sum_j X_(j Nloc)(x) G_j(X) (G_j = block j of the novel-basis coefficients, j < G/2 are the
// nonzero ones) and X_(j Nloc)(alpha_r + u) = X_(j Nloc)(alpha_r) for u in V_mloc (the factors
// s_i, i >= mloc, vanish on V_mloc and are GF(2)-linear), the evaluations at alpha_r + V_mloc are
// those of h_r = sum_j c_(r,j) G_j with c_(r,j) = X_(j Nloc)(phi(r Nloc)) = prod_(bit i of j)
// s_(mloc+i)(phi(r Nloc)) -- small-subfield constants.  So rank r forms h_r (k_shard_top, changeRepr
// included) and runs the top g FFT layers' worth of work as that combination; the remaining layers,
// pointmul and the bottom iFFT layers are local (multipliers from global indices via IdxMap).
//
// Inverse.  The local iFFT gives the product's h_r.  The inner iBasisCvt (index windows inside
// [0,K), K = 16) commutes with iFFT layers >= K (they act on higher bits with multipliers that do not
// depend on the window bits), so it runs locally first.  An all-to-all moves to the "t-sliced"
// layout (rank = index bits [K-g, K)), where the top g iFFT layers and the outer iBasisCvt (windows in
// [K, m)) are local; another all-to-all returns to blocked, where the top Taylor steps of level
// l <= mloc are local and the g steps with l > mloc exchange half a block pairwise.  changeRepr^-1 +
// InterleavedCombine need one tower element from rank r-1.
//
// Data movement is a list of transfers (src rank/buffer/offset -> dst rank/buffer/offset) that every
// rank derives identically; it runs as NCCL grouped send/recv (one process per GPU) or, in the
// single-process simulation with G virtual ranks on one device, as device-to-device copies.
#pragma once
#include <dlfcn.h>

// ---------------------------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------------------------
#define SHARD_MAXG 8       // ranks
#define SHARD_MAXJ 128
#define SHARD_MAXJ_UNR 4   // block words prefetched per point (G <= 8)

struct ShardTopParams {
    const uint64_t* S;   // converted operand, n = (G/2) Nloc words
    uint4* W;            // out: h_r, Nloc tower elements
    const DevTables* tabs;
    uint64_t Nloc;
    int J;               // G/2 blocks
    uint32_t coef[SHARD_MAXJ];
};

// W[i] = sum_j coef_j * psi(S[j Nloc + i])   (coef_j < 2^32: M4R-4 tables, psi: M4R-8 table)
__global__ void __launch_bounds__(256) k_shard_top(ShardTopParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint32_t* tabs = reinterpret_cast<uint32_t*>(smem_raw);
    uint4* psit = reinterpret_cast<uint4*>(tabs + p.J * 128);
    for (int i = threadIdx.x; i < p.J * 8; i += blockDim.x) build_tab_row(tabs + (i >> 3) * 128, p.coef[i >> 3], i & 7, p.tabs->wt);
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) psit[i] = p.tabs->psi64[i];
    __syncthreads();
    const uint32_t tabs_sa = (uint32_t)__cvta_generic_to_shared(tabs);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.Nloc; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 acc = make_uint4(0, 0, 0, 0);
        uint64_t ws[SHARD_MAXJ_UNR];   // the J block words of this point, loaded up front
#pragma unroll
        for (int j = 0; j < SHARD_MAXJ_UNR; j++) ws[j] = j < p.J ? p.S[j * p.Nloc + i] : 0ull;
        for (int j = 0; j < p.J; j++) {
            const uint64_t w = j < SHARD_MAXJ_UNR ? ws[j] : p.S[j * p.Nloc + i];
            uint4 v = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int ch = 0; ch < 8; ch++) v = xor4(v, psit[ch * 256 + ((w >> (8 * ch)) & 255)]);
            if (j == 0) {   // c_(r,0) = X_0 = 1
                acc = xor4(acc, v);
                continue;
            }
            const uint32_t t = tabs_sa + j * 512u;
            acc.x ^= m4r4_word_sa(t, v.x); acc.y ^= m4r4_word_sa(t, v.y);
            acc.z ^= m4r4_word_sa(t, v.z); acc.w ^= m4r4_word_sa(t, v.w);
        }
        p.W[i] = acc;
    }
}

// Same result with the constants folded into the changeRepr tables: T_j[ch][x] = c_j (x) psi(x << 8 ch)
// (both maps are GF(2)-linear), so a point costs J x 8 table reads instead of J x 8 + (J-1) x 32.
// Tables in shared memory (J x 32 KB, J <= 4), built per CTA from psi64 and the c_j M4R-4 rows.
#define SHARD_TOP2_THREADS 512
__global__ void __launch_bounds__(SHARD_TOP2_THREADS) k_shard_top2(ShardTopParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint4* T = reinterpret_cast<uint4*>(smem_raw);                 // [J][8 x 256]
    uint32_t* ct = reinterpret_cast<uint32_t*>(T + p.J * 2048);     // [J][128] M4R-4 rows of c_j
    for (int i = threadIdx.x; i < p.J * 8; i += blockDim.x) build_tab_row(ct + (i >> 3) * 128, p.coef[i >> 3], i & 7, p.tabs->wt);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) T[i] = p.tabs->psi64[i];   // j = 0: c_0 = 1
    __syncthreads();
    const uint32_t ct_sa = (uint32_t)__cvta_generic_to_shared(ct);
    for (int i = threadIdx.x; i < (p.J - 1) * 2048; i += blockDim.x) {
        const int j = 1 + i / 2048, e = i % 2048;
        const uint4 v = T[e];
        const uint32_t t = ct_sa + j * 512u;
        T[j * 2048 + e] = make_uint4(m4r4_word_sa(t, v.x), m4r4_word_sa(t, v.y), m4r4_word_sa(t, v.z), m4r4_word_sa(t, v.w));
    }
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.Nloc; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t ws[SHARD_MAXJ_UNR];
#pragma unroll
        for (int j = 0; j < SHARD_MAXJ_UNR; j++) ws[j] = j < p.J ? p.S[j * p.Nloc + i] : 0ull;
        uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < SHARD_MAXJ_UNR; j++) {
            if (j >= p.J) break;
            const uint64_t w = ws[j];
            if (!w) continue;
            const uint4* tj = T + j * 2048;
#pragma unroll
            for (int ch = 0; ch < 8; ch++) acc = xor4(acc, tj[ch * 256 + ((w >> (8 * ch)) & 255)]);
        }
        p.W[i] = acc;
    }
}

// blocked <-> t-sliced packing.  Element i of a blocked block goes to rank q = bits [K-g, K) of i,
// at position j = (i & (2^(K-g)-1)) | ((i >> K) << (K-g)) of the chunk for q (chunks of Nloc/G).
__device__ __forceinline__ uint64_t pack_src(uint64_t q, uint64_t j, int Kg, int K) {
    return (j & ((1ull << Kg) - 1)) | (q << Kg) | ((j >> Kg) << K);
}
__global__ void k_pack(const uint4* __restrict__ H, uint4* __restrict__ X, uint64_t Nloc, int g, int K, int unpack) {
    const uint64_t chunk = Nloc >> g;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < Nloc; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = t / chunk, j = t - q * chunk;
        const uint64_t i = pack_src(q, j, K - g, K);
        if (unpack) ((uint4*)H)[i] = X[t];
        else X[t] = H[i];
    }
}

// Peer-memory all-to-all fused with the (un)packing (SURVEY §8e "exchange fused with compute"):
//   pull-pack, rank q:   T[r chunk + j] = W_r[pack_src(q, j)]     (every rank r's blocked W)
//   pull-unpack, rank r: W[pack_src(q, j)] = T_q[r chunk + j]     (every rank q's t-sliced T)
// src[] are the G ranks' buffers (IPC-mapped peers over NVLink, or the virtual ranks of the simulation).
struct PullParams {
    const uint4* src[SHARD_MAXG];
    uint4* dst;
    uint64_t chunk;
    int me, G, Kg, K;
};
__global__ void k_pull_pack(PullParams p) {
    const uint64_t total = p.chunk * p.G;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const int r = (int)(t / p.chunk);
        const uint64_t j = t - (uint64_t)r * p.chunk;
        p.dst[t] = p.src[r][pack_src((uint64_t)p.me, j, p.Kg, p.K)];
    }
}
__global__ void k_pull_unpack(PullParams p) {
    const uint64_t total = p.chunk * p.G;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const int q = (int)(t / p.chunk);
        const uint64_t j = t - (uint64_t)q * p.chunk;
        p.dst[pack_src((uint64_t)q, j, p.Kg, p.K)] = p.src[q][(uint64_t)p.me * p.chunk + j];
    }
}

// f[i] ^= src[i], i in [lo, hi)
__global__ void k_xor_range(uint4* __restrict__ f, const uint4* __restrict__ src, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < hi; i += (uint64_t)gridDim.x * blockDim.x)
        f[i] = xor4(f[i], src[i]);
}

// ---------------------------------------------------------------------------------------------
// NCCL, loaded at run time (no link-time dependency; whichever libnccl.so.2 the process has)
// ---------------------------------------------------------------------------------------------
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
struct NcclApi {
    void* h = nullptr;
    int (*GetUniqueId)(nccl_uid_t*);
    int (*CommInitRank)(nccl_comm_t*, int, nccl_uid_t, int);
    int (*CommDestroy)(nccl_comm_t);
    int (*AllGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t);
    int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t);
    int (*Send)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t);
    int (*Recv)(void*, size_t, int, int, nccl_comm_t, cudaStream_t);
    int (*GroupStart)();
    int (*GroupEnd)();
    const char* (*GetErrorString)(int);
    int (*CommGetAsyncError)(nccl_comm_t, int*);   // failure surfacing
    int (*CommAbort)(nccl_comm_t);
};
static const int NCCL_UINT8 = 1;   // ncclUint8 in the ncclDataType_t enum
static const int NCCL_INT32 = 2;   // ncclInt32
static const int NCCL_SUM = 0, NCCL_MIN = 3;   // ncclRedOp_t
static NcclApi g_nccl;
static std::string nccl_load() {
    if (g_nccl.h) return "";
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return std::string("cannot load libnccl.so.2: ") + dlerror();
#define NCCL_SYM(field, name)                                   \
    *(void**)(&g_nccl.field) = dlsym(h, name);                  \
    if (!g_nccl.field) return std::string("missing NCCL symbol ") + name;
    NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    NCCL_SYM(CommInitRank, "ncclCommInitRank");
    NCCL_SYM(CommDestroy, "ncclCommDestroy");
    NCCL_SYM(AllGather, "ncclAllGather");
    NCCL_SYM(AllReduce, "ncclAllReduce");
    NCCL_SYM(Send, "ncclSend");
    NCCL_SYM(Recv, "ncclRecv");
    NCCL_SYM(GroupStart, "ncclGroupStart");
    NCCL_SYM(GroupEnd, "ncclGroupEnd");
    NCCL_SYM(GetErrorString, "ncclGetErrorString");
    NCCL_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    NCCL_SYM(CommAbort, "ncclCommAbort");
#undef NCCL_SYM
    g_nccl.h = h;
    return "";
}

struct gf2x_comm_s {
    int nranks, rank, device;
    nccl_comm_t comm;
    void* ws;          // per-communicator workspace (grown on demand)
    size_t ws_bytes;
    // peer-memory exchange: every rank's workspace mapped into this process (CUDA IPC over NVLink);
    // p2p = 0 falls back to NCCL grouped send/recv
    int p2p;
    void* peer_ws[SHARD_MAXG];
    int* d_sync;       // 1 int (stream-ordered barrier = NCCL all-reduce of it) + IPC handle staging
    int aborted;       // the NCCL communicator was aborted (async error, timeout or gf2x_comm_abort)
    std::string abort_reason;
    // host mode (gf2x_comm_init_host): no NCCL; barriers and the IPC-handle exchange go through the caller's
    // host callbacks (e.g. a torch.distributed gloo group), every exchange is a peer-memory pull
    int host = 0;
    gf2x_host_barrier_fn hbar = nullptr;
    gf2x_host_allgather_fn hag = nullptr;
    void* huser = nullptr;
};

static const int NCCL_IN_PROGRESS = 7;   // ncclInProgress (non-blocking communicators): not an error

static void comm_abort(gf2x_comm_s* c, const std::string& why) {
    if (c->aborted) return;
    c->aborted = 1;
    c->abort_reason = why;
    if (g_nccl.h && c->comm) g_nccl.CommAbort(c->comm);   // unblocks NCCL kernels waiting for a dead peer
    c->comm = nullptr;
}

// ncclCommGetAsyncError: an asynchronous NCCL failure (a peer died, a network error) aborts the
// communicator, so that the stream-ordered barriers of the exchange cannot hang forever
static gf2x_status comm_check(gf2x_comm_s* c) {
    if (c->aborted) return fail(GF2X_ENCCL, "communicator aborted: " + c->abort_reason);
    if (c->host) return GF2X_OK;
    int async = 0;
    int rc = g_nccl.CommGetAsyncError(c->comm, &async);
    if (rc || (async && async != NCCL_IN_PROGRESS)) {
        const int e = rc ? rc : async;
        comm_abort(c, std::string("NCCL asynchronous error: ") + g_nccl.GetErrorString(e));
        return fail(GF2X_ENCCL, c->abort_reason);
    }
    return GF2X_OK;
}

// ---------------------------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------------------------
// workspace buffers (SB_A..SB_HALO) and the caller's input shards (SB_INA, SB_INB: sources only)
// SB_CA, SB_CB: this rank's input shards copied into the workspace (the peer-memory gather reads them)
enum ShardBuf { SB_A = 0, SB_B, SB_W, SB_T, SB_X, SB_HALO, SB_CA, SB_CB, SB_COUNT, SB_INA = SB_COUNT, SB_INB, SB_ALL };

struct RankCtx {
    int r;
    const uint64_t* a_shard;
    const uint64_t* b_shard;
    uint64_t* c_shard;
    unsigned char* buf[SB_ALL];
};

struct Xfer {
    int src, dst;
    ShardBuf sb, db;
    size_t soff, doff, bytes;  // byte offsets
};

struct ShardGeom {
    int G, g, m, mloc, K, p;
    uint64_t n, N, Nloc;
    std::vector<CvtPass> cvt_fwd, inner, outer, top_local;
    std::vector<int> top_cross;  // levels l > mloc, ascending
    std::vector<FftPass> fft;
    Plan lp;                     // local plan (batch 1, N = Nloc) for the FFT launches
    size_t off[SB_COUNT], bytes;
};

static gf2x_status shard_geom(uint64_t bits, int G, ShardGeom& S) {
    if (G < 2 || (G & (G - 1))) return fail(GF2X_EINVAL, "nranks must be a power of two >= 2");
    S.G = G;
    S.g = 0;
    while ((1 << S.g) < G) S.g++;
    S.n = (bits + 63) / 64;
    if (S.n == 0 || (S.n & (S.n - 1))) return fail(GF2X_EINVAL, "sharded multiply needs ceil(bits/64) a power of two");
    S.p = ceil_log2_u64(S.n);
    S.m = S.p + 1;
    if (S.m > 32) return fail(GF2X_ETOOBIG, "FFT size exceeds 2^32 points");
    S.K = 1;
    while (2 * S.K <= S.m - 1) S.K *= 2;
    S.mloc = S.m - S.g;
    if (S.mloc < S.K || S.mloc < BOT_B_MAX + 6 || S.K < S.g)
        return fail(GF2X_EINVAL, "operands too small for this many ranks (need m - log2 G >= max(K, 12))");
    S.N = 1ull << S.m;
    S.Nloc = S.N >> S.g;
    S.cvt_fwd = plan_cvt(S.p, 8);
    std::vector<CvtOp> inner, outer, top_local;
    cvt_ops(S.K, 0, inner);
    cvt_ops(S.m - S.K, S.K, outer);
    for (auto& o : outer) o.lg -= S.g;   // t-sliced layout: global bits >= K sit g lower
    for (int l = S.mloc; l >= S.K + 1; --l) top_local.push_back({l, S.K});
    S.inner = plan_cvt_ops(inner, S.mloc, 16);
    S.outer = plan_cvt_ops(outer, S.mloc, 16);
    S.top_local = plan_cvt_ops(top_local, S.mloc, 16);
    S.top_cross.clear();
    for (int l = S.mloc + 1; l <= S.m; l++) S.top_cross.push_back(l);
    S.fft = plan_fft(S.mloc);
    S.lp = Plan();
    S.lp.na = S.lp.nb = S.Nloc / 2;
    S.lp.N = S.Nloc;
    S.lp.batch = 1;
    S.lp.m = S.mloc;
    S.lp.ma = S.lp.mb = S.mloc - 1;
    S.lp.fft = S.fft;
    // per-rank buffers
    size_t o = 0;
    S.off[SB_A] = o; o = align256(o + S.n * 8);
    S.off[SB_B] = o; o = align256(o + S.n * 8);
    S.off[SB_W] = o; o = align256(o + (2 * S.Nloc + 2048) * 16);   // Wa | Wb | bottom pad
    S.off[SB_T] = o; o = align256(o + S.Nloc * 16);
    S.off[SB_X] = o; o = align256(o + S.Nloc * 16);
    S.off[SB_HALO] = o; o = align256(o + 16);
    S.off[SB_CA] = o; o = align256(o + S.n / G * 8);
    S.off[SB_CB] = o; o = align256(o + S.n / G * 8);
    S.bytes = o;
    return GF2X_OK;
}

// s_k(phi(b)) for any b < 2^32 on the host: XOR of S[k][j] = s_k(v_j) over the set bits j of b
// (S[k][j] = 0 for j < k, S[k][k] = s_k(v_k) = 1 by Prop. 1)
static uint32_t host_s_eval(const DevTables* T, int k, uint64_t b) {
    uint32_t c = 0;
    for (int j = 0; j < 32; j++)
        if ((b >> j) & 1) c ^= T->S[k * 32 + j];
    return c;
}

struct ShardExec {
    bool sim;
    gf2x_comm_s* comm;   // NCCL mode
    cudaStream_t st;
    std::vector<RankCtx>* ranks;   // all ranks (sim) or the local one (NCCL)
    bool p2p = false;              // pull from peer memory (sim: the virtual ranks' buffers; NCCL: IPC-mapped)
    unsigned char* peer[SHARD_MAXG] = {};   // p2p, NCCL mode: every rank's workspace base
    const size_t* off = nullptr;   // buffer offsets in a workspace (ShardGeom::off)
    // pointer to rank r's buffer b (p2p)
    unsigned char* rbuf(int r, ShardBuf b) {
        if (sim) return (*ranks)[r].buf[b];
        if (r == comm->rank) return (*ranks)[0].buf[b];
        return peer[r] + off[b];
    }
    // stream-ordered barrier of all ranks: every rank's work enqueued before it has finished when any
    // rank's work enqueued after it starts (NCCL all-reduce of one int); nothing to do in the simulation
    gf2x_status barrier() {
        if (sim) return GF2X_OK;
        if (comm->host) {   // host barrier: this rank's enqueued work is complete, then the caller's barrier
            CUDA_TRY(cudaStreamSynchronize(st));
            if (comm->hbar(comm->huser) != 0) return fail(GF2X_ENCCL, "host barrier callback failed");
            return GF2X_OK;
        }
        int rc = g_nccl.AllReduce(comm->d_sync, comm->d_sync, 1, NCCL_INT32, NCCL_SUM, comm->comm, st);
        if (rc) return fail(GF2X_ENCCL, std::string("NCCL barrier: ") + g_nccl.GetErrorString(rc));
        return GF2X_OK;
    }
    gf2x_status run(const std::vector<Xfer>& xs) {
        if (p2p) {   // every destination pulls its transfers from the source's memory
            gf2x_status s = barrier();
            if (s != GF2X_OK) return s;
            for (const Xfer& x : xs) {
                if (!owns(x.dst)) continue;
                ShardBuf sb = x.sb;
                if (!sim && sb == SB_INA) sb = SB_CA;   // peers' input shards are read from their copies
                if (!sim && sb == SB_INB) sb = SB_CB;
                const unsigned char* src = (sim || x.src == comm->rank) ? local(x.src).buf[sb] + x.soff
                                                                         : rbuf(x.src, sb) + x.soff;
                cudaError_t e = cudaMemcpyAsync(local(x.dst).buf[x.db] + x.doff, src, x.bytes, cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("shard pull: ") + cudaGetErrorString(e));
            }
            return barrier();   // the sources may be overwritten once every pull has finished
        }
        if (sim) {
            for (const Xfer& x : xs) {
                RankCtx& s = (*ranks)[x.src];
                RankCtx& d = (*ranks)[x.dst];
                cudaError_t e = cudaMemcpyAsync(d.buf[x.db] + x.doff, s.buf[x.sb] + x.soff, x.bytes, cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("shard copy: ") + cudaGetErrorString(e));
            }
            return GF2X_OK;
        }
        RankCtx& me = (*ranks)[0];
        if (comm->host) return fail(GF2X_EINVAL, "host-mode communicator: peer-memory exchanges only");
        int rc = g_nccl.GroupStart();
        for (const Xfer& x : xs) {
            if (rc) break;
            if (x.src == comm->rank && x.dst == comm->rank) {
                cudaError_t e = cudaMemcpyAsync(me.buf[x.db] + x.doff, me.buf[x.sb] + x.soff, x.bytes, cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) rc = -1;
            } else if (x.src == comm->rank) {
                rc = g_nccl.Send(me.buf[x.sb] + x.soff, x.bytes, NCCL_UINT8, x.dst, comm->comm, st);
            } else if (x.dst == comm->rank) {
                rc = g_nccl.Recv(me.buf[x.db] + x.doff, x.bytes, NCCL_UINT8, x.src, comm->comm, st);
            }
        }
        int rc2 = g_nccl.GroupEnd();
        if (rc || rc2) return fail(GF2X_ENCCL, std::string("NCCL exchange failed: ") + g_nccl.GetErrorString(rc ? rc : rc2));
        return GF2X_OK;
    }
    RankCtx& local(int r) {
        if (sim) return (*ranks)[r];
        return (*ranks)[0];
    }
    bool owns(int r) const { return sim || r == comm->rank; }
};

// Every exchange of the sharded multiply as transfer lists (host only; every rank derives the same
// lists from (bits, G)).  Byte offsets into the per-rank buffers of ShardGeom.
struct ShardXfers {
    // rank r converts operand r & 1 (0: a, 1: b): gather that operand's shards from every rank into A,
    // then hand the converted operand to the partner rank r ^ 1 (its B)
    std::vector<Xfer> gather;
    std::vector<Xfer> xchg;
    std::vector<Xfer> a2a_fwd;                 // blocked -> t-sliced: rank r's chunk q -> rank q's T chunk r
    std::vector<Xfer> a2a_back;                // t-sliced -> blocked: rank q's T chunk r -> rank r's X chunk q
    std::vector<std::vector<Xfer>> cross;      // one per level in ShardGeom::top_cross (ascending)
    std::vector<Xfer> halo;                    // last tower element of rank r-1 -> rank r
};
static void shard_xfers(const ShardGeom& S, ShardXfers& X) {
    const int G = S.G;
    const uint64_t chunk = S.Nloc >> S.g, Nloc = S.Nloc;
    X.gather.clear(); X.xchg.clear(); X.a2a_fwd.clear(); X.a2a_back.clear(); X.cross.clear(); X.halo.clear();
    const uint64_t sb = S.n / G * 8;   // bytes of an operand shard
    for (int r = 0; r < G; r++)
        for (int q = 0; q < G; q++) X.gather.push_back({q, r, (r & 1) ? SB_INB : SB_INA, SB_A, 0, q * sb, sb});
    for (int r = 0; r < G; r++) X.xchg.push_back({r, r ^ 1, SB_A, SB_B, 0, 0, S.n * 8});
    for (int r = 0; r < G; r++)
        for (int q = 0; q < G; q++) X.a2a_fwd.push_back({r, q, SB_X, SB_T, q * chunk * 16, r * chunk * 16, chunk * 16});
    for (int q = 0; q < G; q++)
        for (int r = 0; r < G; r++) X.a2a_back.push_back({q, r, SB_T, SB_X, r * chunk * 16, q * chunk * 16, chunk * 16});
    for (int l : S.top_cross) {
        const int Sb = 1 << (l - S.mloc);          // blocks per segment
        const uint64_t u = 1ull << (l - 1 - S.K);  // window unit
        std::vector<Xfer> xs;
        for (int base = 0; base < G; base += Sb) {
            for (int p = 0; p < Sb / 2; p++) {
                // phase B^-1 sources for rank base+p: t + d = t + h - u
                xs.push_back({base + p + Sb / 2, base + p, SB_W, SB_X, 0, u * 16, (Nloc - u) * 16});
                if (p >= 1) xs.push_back({base + p + Sb / 2 - 1, base + p, SB_W, SB_X, (Nloc - u) * 16, 0, u * 16});
            }
            // phase A^-1 sources: [2h-u, 2h) -> rank base + Sb/2, targets [0, u)
            xs.push_back({base + Sb - 1, base + Sb / 2, SB_W, SB_T, (Nloc - u) * 16, 0, u * 16});
        }
        X.cross.push_back(xs);
    }
    for (int r = 1; r < G; r++) X.halo.push_back({r - 1, r, SB_W, SB_HALO, (Nloc - 1) * 16, 0, 16});
}

// debug_stage (simulation only): 1 = stop after the forward FFT (copy every rank's Wa block to dbg),
// 5 = stop after the whole iBasisCvt (copy the blocked W blocks).  dbg: N tower elements.
static gf2x_status run_sharded(const ShardGeom& S, ShardExec& X, DeviceState* ds, const DevTables* host_tabs, uint64_t bits,
                               int debug_stage = 0, uint4* dbg = nullptr) {
    gf2x_status s;
    const int G = S.G, g = S.g, smc = ds->sm_count;
    ShardXfers XF;
    shard_xfers(S, XF);
    cudaStream_t st = X.st;
    const uint64_t Nloc = S.Nloc, chunk = Nloc >> g;
    std::vector<int> mine;
    for (int r = 0; r < G; r++)
        if (X.owns(r)) mine.push_back(r);
    auto last = [&](const char* what) -> gf2x_status {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
        return GF2X_OK;
    };
    // ---- gather: rank r assembles operand r & 1 (a for even ranks, b for odd ones) and converts only that
    // one (the forward conversion is a whole-operand transform done redundantly; splitting it between
    // partner ranks halves it), then partners swap their converted operands
    if (X.p2p && !X.sim)   // this rank's input shards into its workspace, where the peers pull them from
        for (int r : mine) {
            RankCtx& R = X.local(r);
            CUDA_TRY(cudaMemcpyAsync(R.buf[SB_CA], R.a_shard, S.n / G * 8, cudaMemcpyDeviceToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(R.buf[SB_CB], R.b_shard, S.n / G * 8, cudaMemcpyDeviceToDevice, st));
        }
    if ((s = X.run(XF.gather)) != GF2X_OK) return s;
    for (int r : mine) {
        uint64_t* A = (uint64_t*)X.local(r).buf[SB_A];
        if (!S.cvt_fwd.empty() && top_rowbits(S.cvt_fwd[0], S.p) >= 0 && !env_flag("GF2X_NO_FUSED_SPLIT")) {
            // Split (the mask of the last word) fused into the top Taylor pass, in place (k_cvt_top)
            const CvtSrc src{A, A, 1, S.n, bits};
            if ((s = run_cvt<uint64_t>(S.cvt_fwd, A, S.p, 1, false, smc, st, &src)) != GF2X_OK) return s;
            continue;
        }
        { ProfScope ps("k_prep", 16.0 * S.n, st); k_prep<<<grid_for(S.n, 256, smc, 8), 256, 0, st>>>(A, S.n, bits, S.p, 1, A); }
        if ((s = last("shard prep")) != GF2X_OK) return s;
        if ((s = run_cvt<uint64_t>(S.cvt_fwd, A, S.p, 1, false, smc, st)) != GF2X_OK) return s;
    }
    if ((s = X.run(XF.xchg)) != GF2X_OK) return s;
    // ---- combine into h_r (changeRepr included), local FFT
    for (int r : mine) {
        RankCtx& R = X.local(r);
        uint64_t* A = (uint64_t*)R.buf[(r & 1) ? SB_B : SB_A];   // converted a
        uint64_t* B = (uint64_t*)R.buf[(r & 1) ? SB_A : SB_B];   // converted b
        uint4* W = (uint4*)R.buf[SB_W];
        ShardTopParams tp;
        tp.tabs = ds->tabs;
        tp.Nloc = Nloc;
        tp.J = G / 2;
        const uint64_t ar = (uint64_t)r * Nloc;   // alpha_r = phi(r Nloc)
        for (int j = 0; j < tp.J; j++) {
            gf2x_host::u128 c = 1;
            for (int i = 0; i < g; i++)
                if ((j >> i) & 1) c = gf2x_host::tower_mul(c, (gf2x_host::u128)host_s_eval(host_tabs, S.mloc + i, ar));
            tp.coef[j] = (uint32_t)c;
        }
        // composed tables (k_shard_top2) while J x 32 KB fits; the M4R-4 version beyond (J > 4 never at G <= 8)
        const bool top2 = tp.J <= SHARD_MAXJ_UNR && !env_flag("GF2X_SHARD_TOP1");
        const size_t sm = top2 ? (size_t)tp.J * (2048 * 16 + 512) : (size_t)tp.J * 512 + 8 * 256 * 16;
        if (top2) cudaFuncSetAttribute(k_shard_top2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        else cudaFuncSetAttribute(k_shard_top, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int o = 0; o < 2; o++) {
            tp.S = o ? B : A; tp.W = W + o * Nloc;
            ProfScope ps("k_shard_top", 8.0 * tp.J * Nloc + 16.0 * Nloc, st);
            if (top2) k_shard_top2<<<grid_for(Nloc, SHARD_TOP2_THREADS, smc, 1), SHARD_TOP2_THREADS, sm, st>>>(tp);
            else k_shard_top<<<grid_for(Nloc, 256, smc, 4), 256, sm, st>>>(tp);
        }
        if ((s = last("shard top")) != GF2X_OK) return s;
        // ---- local FFT layers [6, mloc) of both operands, bottom kernel, local iFFT layers
        const IdxMap map{S.mloc, g, (uint32_t)r};
        const size_t nd = S.fft.size() - 1;
        for (size_t i = 0; i < nd; i++)
            if ((s = launch_fft(S.fft[i], false, false, W, Nloc, W, S.lp, ds, st, 2, map)) != GF2X_OK) return s;
        BottomParams bp;
        bp.A = W; bp.B = W + Nloc;
        bp.total = Nloc;
        bp.ntiles = (Nloc + (1ull << BT_BITS) - 1) >> BT_BITS;
        bp.m = S.mloc; bp.L = S.fft.back().layers; bp.mode = debug_stage == 1 ? 1 : 7;
        bp.map = map;
        {
            ProfScope ps("k_bottom", 48.0 * Nloc, st, bottom_alu_ops(bp));
            bottom_launch(bp, smc, st);
        }
        if ((s = last("shard bottom")) != GF2X_OK) return s;
        if (debug_stage == 1) {
            cudaMemcpyAsync(dbg + r * Nloc, W, Nloc * 16, cudaMemcpyDeviceToDevice, st);
            continue;
        }
        for (size_t i = nd; i-- > 0;)
            if ((s = launch_fft(S.fft[i], true, false, W, Nloc, W, S.lp, ds, st, 1, map)) != GF2X_OK) return s;
        // ---- inner iBasisCvt (windows in [0, K)) locally, then pack by destination rank
        if ((s = run_cvt<uint4>(S.inner, W, S.mloc, 1, true, smc, st)) != GF2X_OK) return s;
        if (!X.p2p) {
            ProfScope ps("k_pack", 32.0 * Nloc, st);
            k_pack<<<grid_for(Nloc, 256, smc, 8), 256, 0, st>>>(W, (uint4*)R.buf[SB_X], Nloc, g, S.K, 0);
        }
        if ((s = last("shard pack")) != GF2X_OK) return s;
    }
    if (debug_stage == 1) return GF2X_OK;
    // ---- all-to-all: rank r's chunk q -> rank q's T at chunk r (peer memory: pulled and packed in one kernel)
    auto pull = [&](bool unpack) -> gf2x_status {
        gf2x_status s2 = X.barrier();
        if (s2 != GF2X_OK) return s2;
        for (int q : mine) {
            PullParams pp;
            for (int r = 0; r < G; r++) pp.src[r] = (const uint4*)X.rbuf(r, unpack ? SB_T : SB_W);
            pp.dst = (uint4*)X.local(q).buf[unpack ? SB_W : SB_T];
            pp.chunk = chunk; pp.me = q; pp.G = G; pp.Kg = S.K - g; pp.K = S.K;
            ProfScope ps(unpack ? "k_pull_unpack" : "k_pull_pack", 32.0 * Nloc, st);
            if (unpack) k_pull_unpack<<<grid_for(Nloc, 256, smc, 8), 256, 0, st>>>(pp);
            else k_pull_pack<<<grid_for(Nloc, 256, smc, 8), 256, 0, st>>>(pp);
            if ((s2 = last("shard pull")) != GF2X_OK) return s2;
        }
        return X.barrier();
    };
    if (X.p2p) { if ((s = pull(false)) != GF2X_OK) return s; }
    else if ((s = X.run(XF.a2a_fwd)) != GF2X_OK) return s;
    // ---- t-sliced: top g iFFT layers, outer iBasisCvt
    for (int q : mine) {
        RankCtx& R = X.local(q);
        uint4* T = (uint4*)R.buf[SB_T];
        const IdxMap tmap{S.K - g, g, (uint32_t)q};
        FftPass top{6, S.mloc - g, S.mloc, false, 0};
        if ((s = launch_fft(top, true, false, T, Nloc, T, S.lp, ds, st, 1, tmap)) != GF2X_OK) return s;
        if ((s = run_cvt<uint4>(S.outer, T, S.mloc, 1, true, smc, st)) != GF2X_OK) return s;
    }
    // ---- all-to-all back: rank q's T chunk r -> rank r's X chunk q, unpack
    if (X.p2p) { if ((s = pull(true)) != GF2X_OK) return s; }
    else if ((s = X.run(XF.a2a_back)) != GF2X_OK) return s;
    for (int r : mine) {
        RankCtx& R = X.local(r);
        uint4* W = (uint4*)R.buf[SB_W];
        if (!X.p2p) {
            ProfScope ps("k_pack", 32.0 * Nloc, st);
            k_pack<<<grid_for(Nloc, 256, smc, 8), 256, 0, st>>>(W, (uint4*)R.buf[SB_X], Nloc, g, S.K, 1);
        }
        if ((s = last("shard unpack")) != GF2X_OK) return s;
        if ((s = run_cvt<uint4>(S.top_local, W, S.mloc, 1, true, smc, st)) != GF2X_OK) return s;
    }
    // ---- top Taylor steps spanning ranks, ascending level (inverse order)
    for (size_t li = 0; li < S.top_cross.size(); li++) {
        const int l = S.top_cross[li];
        const int Sb = 1 << (l - S.mloc);          // blocks per segment
        const uint64_t u = 1ull << (l - 1 - S.K);  // window unit
        if ((s = X.run(XF.cross[li])) != GF2X_OK) return s;
        for (int r : mine) {
            RankCtx& R = X.local(r);
            uint4* W = (uint4*)R.buf[SB_W];
            const int p = r % Sb;
            if (p < Sb / 2) {
                const uint64_t lo = (p == 0) ? u : 0;
                ProfScope ps("k_xor_range", 48.0 * (Nloc - lo), st);
                k_xor_range<<<grid_for(Nloc - lo, 256, smc, 8), 256, 0, st>>>(W, (uint4*)R.buf[SB_X], lo, Nloc);
            } else if (p == Sb / 2) {
                ProfScope ps("k_xor_range", 48.0 * u, st);
                k_xor_range<<<grid_for(u, 256, smc, 8), 256, 0, st>>>(W, (uint4*)R.buf[SB_T], 0, u);
            }
            if ((s = last("shard cross step")) != GF2X_OK) return s;
        }
    }
    if (debug_stage == 5) {
        for (int r : mine) cudaMemcpyAsync(dbg + r * Nloc, X.local(r).buf[SB_W], Nloc * 16, cudaMemcpyDeviceToDevice, st);
        return GF2X_OK;
    }
    // ---- halo: last element of rank r-1 -> rank r; changeRepr^-1 + InterleavedCombine
    if ((s = X.run(XF.halo)) != GF2X_OK) return s;
    for (int r : mine) {
        RankCtx& R = X.local(r);
        const uint4* halo = r ? (const uint4*)R.buf[SB_HALO] : nullptr;
        if (Nloc % IB_TILE == 0) {
            ProfScope ps("k_ipsi_bs", 24.0 * Nloc, st);
            k_ipsi_bs<false><<<grid_for(Nloc / IB_TILE, 1, smc, 2), IB_THREADS, 6 * IB_TILE * 4, st>>>((const uint4*)R.buf[SB_W], ds->tabs,
                                                                                                 Nloc, 1, R.c_shard, halo, Nloc);
        } else {
            ProfScope ps("k_ipsi_combine", 24.0 * Nloc, st);
            k_ipsi_combine<<<grid_for(Nloc, 256, smc, 2), 256, 16 * 256 * 16, st>>>((const uint4*)R.buf[SB_W], ds->tabs, Nloc,
                                                                                    Nloc, 1, R.c_shard, halo);
        }
        if ((s = last("shard combine")) != GF2X_OK) return s;
    }
    return GF2X_OK;
}
