// gf2x.cu -- sm_100a implementation of the C ABI in include/gf2x.h.
//
// Pipeline (Alg. 5), per product of n_a x n_b 64-bit words, N = 2^m points:
//   k_prep          Split: copy + mask words into the conversion scratch S (u64)
//   k_cvt_*         BasisCvt (Alg. 3 P:518-539 / Alg. 2) on 64-bit words, in place in S
//   k_fft2<psi>     changeRepr (§4.3) fused into the first FFT_LCH pass (Alg. 1)
//   k_fft2          FFT_LCH layers >= 6 (tiles of layers through shared memory, M4R-4 tables)
//   k_bottom        FFT_LCH layers < 6 of a and b, pointmul, iFFT_LCH layers < 6,
//                   fused and bit-sliced
//   k_fft2<inverse> iFFT_LCH layers >= 6
//   k_cvt_*         iBasisCvt on 128-bit tower elements
//   k_ipsi_bs       changeRepr back + InterleavedCombine, bit-sliced
//                   (k_ipsi_combine: table-driven fallback)
// w = 128 (TGF(2^256)): w128.cuh.  Alg. 4: alg4.cuh.  Multi-GPU: shard.cuh.
// Every step runs in these kernels; the host only plans passes and enqueues launches.
//
// Diagnostic / A-B knobs (environment, read once per process; defaults are the measured best):
//   GF2X_DEBUG_PLAN=1    print every plan (conversion and FFT passes) to stderr
//   GF2X_NO_RB=1         CVT(8) nodes as shared-memory tile passes instead of register-blocked passes
//   GF2X_NO_RES8=1       K=8 Taylor runs as tile passes instead of residue-class passes
//   (every flag: unset, empty or "0" = off)
//   GF2X_NO_IPSI_BS=1    table-driven changeRepr^-1 + combine instead of the bit-sliced kernel
//   GF2X_FFT_C=c         column bits of the non-first FFT passes shorter than 6 layers (default 6)
//   GF2X_BOT_B=L         layers in the bit-sliced bottom kernel (default 6; 5 for m <= 10)
//   GF2X_MAXR=R          maximum FFT layers per table pass below the changeRepr pass (default 7)
//   GF2X_NO_W2_BS=1      w = 128: table-driven changeRepr_256 / changeRepr_256^-1 instead of bit-sliced
//   GF2X_SHARD_NCCL=1    sharded multiply: NCCL send/recv instead of peer memory (read when a
//                        communicator's workspace is allocated)
//   GF2X_SHARD_LISTS=1   sharded simulation: run the transfer lists as copies (the NCCL path's data
//                        movement) instead of the peer-memory pulls (read per call)
//   GF2X_SHARD_TOP1=1    sharded forward: M4R-4 constant products after changeRepr instead of the composed
//                        changeRepr tables (k_shard_top instead of k_shard_top2)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <ctype.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gf2x.h"
#include "field_host.h"
#include "gf2x_device.cuh"
#include "bitslice_gen.cuh"

using namespace gf2x_dev;

// =============================================================================================
// Constant tables (built on the host by field_host.h, uploaded once per device)
// =============================================================================================
struct DevTables {
    uint4 psi64[8 * 256];    // M4R-8 of changeRepr on a 64-bit polynomial-basis block -> tower
    uint4 ipsi[16 * 256];    // M4R-8 of changeRepr^-1: 128-bit tower element -> polynomial basis
    uint32_t wt[7 * 1024];   // M4R-8 of c -> c * v_(4t), t = 1..7 (table-build helper)
    uint32_t S[32 * 32];     // S[k][j] = s_k(v_j): images of the basis under s_k (§4.4)
};

__constant__ uint32_t c_S[32 * 32];


// =============================================================================================
// Multiplier of layer k for block base b (index within one product): s_k(phi_v(b)) is GF(2)-linear
// in b, so it is the XOR of S[k][j] over the set bits j > k of b (bits <= k of a block base are 0).
// =============================================================================================
__device__ __forceinline__ uint32_t layer_const(int k, uint32_t b) {
    uint32_t c = 0;
    b >>= (k + 1);
    int j = k + 1;
    while (b) {
        if (b & 1) c ^= c_S[k * 32 + j];
        b >>= 1;
        ++j;
    }
    return c;
}

// =============================================================================================
// Index map from a local element index to the global index that fixes the FFT multipliers (used by
// the sharded multiply, where a rank holds a block or a "t-sliced" part of the index space):
//   global = (li & (2^pos - 1)) | (val << pos) | ((li >> pos) << (pos + bits)),
// and a local layer lk maps to global layer lk (+ bits if lk >= pos).  Identity when bits = 0.
// =============================================================================================
struct IdxMap {
    int pos, bits;
    uint32_t val;
};
__device__ __forceinline__ uint32_t gidx(const IdxMap& M, uint32_t li) {
    if (!M.bits) return li;
    return (li & ((1u << M.pos) - 1)) | (M.val << M.pos) | ((li >> M.pos) << (M.pos + M.bits));
}
__device__ __forceinline__ int glayer(const IdxMap& M, int lk) { return lk >= M.pos ? lk + M.bits : lk; }

// =============================================================================================
// k_prep: Split.  Operand pair p occupies words [p*n, (p+1)*n) of `in`; it is copied to
// S[p * 2^ms ...], masked to `bits`, zero-padded to 2^ms words.
// =============================================================================================
__global__ void k_prep(const uint64_t* __restrict__ in, uint64_t n, uint64_t bits, int ms, uint64_t batch,
                       uint64_t* __restrict__ S) {
    const uint64_t per = 1ull << ms, total = per * batch;
    const uint64_t rem = bits & 63;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = i >> ms, j = i & (per - 1);
        uint64_t w = 0;
        if (j < n) {
            w = in[p * n + j];
            if (j == n - 1 && rem) w &= (1ull << rem) - 1;
        }
        S[i] = w;
    }
}

#include "cvt.cuh"
#include "fft.cuh"

// =============================================================================================
// pointmul: P[i] = A[i] (x) B[i] in TGF(2^128).  Each thread owns 32 consecutive
// elements, bit-sliced in place in shared memory (transpose32 per limb: plane j of limb L = bit j of
// the 32 limbs L).  With a = alpha0 + alpha1 x7, alpha_i = A_2i + A_2i+1 x6 (x6^2 = x6 + v31,
// x7^2 = x7 + v63, v63 = v31 x6), two Karatsuba levels give nine TGF(2^32) products
//   P0=A0B0 P1=A1B1 P01=(A0+A1)(B0+B1) P2=A2B2 P3=A3B3 P23=(A2+A3)(B2+B3)
//   Q0=(A0+A2)(B0+B2) Q1=(A1+A3)(B1+B3) Q01=(A0+A1+A2+A3)(B0+B1+B2+B3)
// and the result limbs
//   R0 = P0 + v31 P1 + v31^2 (P2 + P23)        R1 = P0 + P01 + v31 P23 + v31^2 P3
//   R2 = P0 + Q0 + v31 (P1 + Q1)               R3 = P0 + P01 + Q0 + Q01
// Each product is one generated straight-line bit-sliced Karatsuba (bs_mul32); only one is live
// in registers at a time.
// =============================================================================================
// (limb mask of the factors, limbs receiving r, limbs receiving v31 r, limbs receiving v31^2 r)
__constant__ int c_pm_terms[9][4] = {
    {0x1, 0xF, 0x0, 0x0},   // P0  -> R0 R1 R2 R3
    {0x2, 0x0, 0x5, 0x0},   // P1  -> v31: R0 R2
    {0x3, 0xA, 0x0, 0x0},   // P01 -> R1 R3
    {0x4, 0x0, 0x0, 0x1},   // P2  -> v31^2: R0
    {0x8, 0x0, 0x0, 0x2},   // P3  -> v31^2: R1
    {0xC, 0x0, 0x2, 0x1},   // P23 -> v31: R1, v31^2: R0
    {0x5, 0xC, 0x0, 0x0},   // Q0  -> R2 R3
    {0xA, 0x0, 0x4, 0x0},   // Q1  -> v31: R2
    {0xF, 0x8, 0x0, 0x0},   // Q01 -> R3
};

#include "bottom.cuh"
#include "small.cuh"
#include "tc_experiment.cuh"

// =============================================================================================
// changeRepr^-1 + InterleavedCombine: C_i = psi^-1(P[i]) (deg <= 126),
// out[w] = lo64(C_w) ^ hi64(C_(w-1)), w < n_out = n_a + n_b, C_i = 0 for i >= N.
// =============================================================================================
__device__ __forceinline__ void ipsi_apply(const uint4* __restrict__ tab, uint4 v, uint64_t& lo, uint64_t& hi) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int L = 0; L < 4; L++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc = xor4(acc, tab[(L * 4 + b) * 256 + ((w[L] >> (8 * b)) & 255)]);
    lo = ((uint64_t)acc.y << 32) | acc.x;
    hi = ((uint64_t)acc.w << 32) | acc.z;
}

// halo (sharded multiply): the tower element that precedes P[0] globally (rank r-1's last one), or null
__global__ void __launch_bounds__(256) k_ipsi_combine(const uint4* __restrict__ P, const DevTables* tabs, uint64_t N,
                                                      uint64_t n_out, uint64_t batch, uint64_t* __restrict__ out,
                                                      const uint4* __restrict__ halo) {
    extern __shared__ __align__(16) uint4 itab[];
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) itab[i] = tabs->ipsi[i];
    __syncthreads();
    const uint64_t total = n_out * batch;
    // grid-stride in whole warps so that the shuffle below always sees its neighbour
    for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < total; i0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = i0 + threadIdx.x;
        const bool in = i < total;
        const uint64_t pair = in ? i / n_out : 0, w = in ? i - pair * n_out : 0;
        uint64_t lo = 0, hi = 0;
        if (in && w < N) ipsi_apply(itab, P[pair * N + w], lo, hi);
        uint64_t prev_hi = __shfl_up_sync(0xFFFFFFFFu, hi, 1);
        const int lane = threadIdx.x & 31;
        if (in) {
            if (lane == 0 || w == 0) {
                prev_hi = 0;
                uint64_t l2;
                if (w >= 1 && w - 1 < N) ipsi_apply(itab, P[pair * N + w - 1], l2, prev_hi);
                else if (w == 0 && halo) ipsi_apply(itab, *halo, l2, prev_hi);
            }
            out[i] = lo ^ prev_hi;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Bit-sliced changeRepr^-1 + InterleavedCombine (used when n_out = N and N is a multiple of 4096):
// thread t of a 128-thread CTA owns the 32 consecutive elements 32t..32t+31 of a 4096-element tile.
// Each input limb is transposed into 32 planes (bit j of the 32 elements), the fixed 128x128 GF(2)
// matrix of changeRepr^-1 is applied as 16 generated 32x32 XOR networks (bs_ipsi_O_L, Paar-style
// common-pair elimination: 3457 XOR per 32 elements), and the output planes are transposed back.
// This replaces 16 random 16-byte table lookups per element (bank-conflicted LDS.128).
// Shared memory: limb-planar tile (4 x 4096 words, XOR-swizzled so that a thread's 32-element column
// and a warp's 32 consecutive elements are both conflict-free) + hi64 of every element (2 x 4096 words).
// ---------------------------------------------------------------------------------------------
#define IB_THREADS 128
#define IB_TILE 4096
__device__ __forceinline__ uint32_t ib_swz(uint32_t e) { return e ^ ((e >> 5) & 31); }

// halo (sharded multiply, batch 1): the tower element preceding P[0] globally (rank r-1's last one), or null
// n_write: flat output words written (N batch when n_out = N; n_out <= N for a single product)
// MC (R28): instead of InterleavedCombine, write D = lo64(C) ^ M hi64(C) in the NOVEL basis, where M is
// the shift by one block written in that basis (multiplication by y = X_1):
//     (M h)[j] = h[j-1] ^ [j odd] h[j] ^ [j even, j > 0] h[j + 2^ctz(j) - 1]      (j within its product)
// so that iBasisCvt of the 64-bit D (in place, in `out`) is the product: half the conversion traffic of the
// 128-bit iBasisCvt it replaces.  The partner of a tile-aligned j (ctz >= 12) lies in another tile (thread 0).
__device__ __forceinline__ uint64_t ipsi_hi_global(const uint4 pv, const DevTables* tabs) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {pv.x, pv.y, pv.z, pv.w};
    for (int L = 0; L < 4; L++)
        for (int b = 0; b < 4; b++) acc = xor4(acc, tabs->ipsi[(L * 4 + b) * 256 + ((w[L] >> (8 * b)) & 255)]);
    return ((uint64_t)acc.w << 32) | acc.z;   // (only the high half is needed)
}
template <bool MC>
__global__ void __launch_bounds__(IB_THREADS, 2) k_ipsi_bs(const uint4* __restrict__ P, const DevTables* tabs, uint64_t N,
                                                         uint64_t batch, uint64_t* __restrict__ out,
                                                         const uint4* __restrict__ halo, uint64_t n_write,
                                                         uint64_t n_valid = ~0ull,   // elements >= n_valid read as 0
                                                         int l2pf = 0) {             // L2 prefetch of the next tile
    extern __shared__ __align__(1024) uint32_t ib_smem[];
    uint32_t* S = ib_smem;                    // [4][IB_TILE] limb planes (swizzled)
    uint32_t* H = ib_smem + 4 * IB_TILE;      // [2][IB_TILE] hi64 halves of every element (swizzled)
    __shared__ uint64_t halo_hi, far_hi;
    // the batch is one flat run of products (n_out = N): a tile covers IB_TILE consecutive elements, which
    // may span several small products; an element at a product boundary has no predecessor
    const uint64_t ntiles = (n_write + IB_TILE - 1) / IB_TILE;
    const uint64_t pair = 0;
    const uint32_t t = threadIdx.x;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t w0 = tile * IB_TILE;   // first element / word of the tile (flat)
        const uint4* src = P + w0;
        if (l2pf && t == 0 && (tile + gridDim.x + 1) * IB_TILE <= n_valid && (tile + gridDim.x + 1) * IB_TILE <= n_write)
            bulk_prefetch_l2(P + (tile + gridDim.x) * IB_TILE, IB_TILE * 16);   // the CTA's next tile into L2
        // ---- load (coalesced), limb-planar; 16 loads in flight per thread (the tile is not prefetched: a second
        // 64 KB buffer would halve the occupancy)
#pragma unroll 1
        for (uint32_t e0 = t; e0 < IB_TILE; e0 += 16 * IB_THREADS) {
            uint4 v[16];
#pragma unroll
            for (int u = 0; u < 16; u++)
                v[u] = w0 + e0 + u * IB_THREADS < n_valid ? src[e0 + u * IB_THREADS] : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 16; u++) {
                const uint32_t q = ib_swz(e0 + u * IB_THREADS);
                S[q] = v[u].x; S[IB_TILE + q] = v[u].y; S[2 * IB_TILE + q] = v[u].z; S[3 * IB_TILE + q] = v[u].w;
            }
        }
        // the element before the tile (its hi64 enters the tile's first output word)
        if (t == 0) {
            uint64_t hi = 0;
            const uint64_t jj = w0 & (N - 1);   // N is a power of two
            if (jj != 0 || halo) hi = ipsi_hi_global(jj != 0 ? src[-1] : *halo, tabs);
            halo_hi = hi;
        }
        if (MC && t == 32) {   // (another warp, so that the two table walks overlap)
            // the tile's first word, if tile-aligned inside its product, also takes h[j + 2^ctz(j) - 1]
            const uint64_t jj = w0 & (N - 1);
            const uint64_t d = (1ull << __ffsll((long long)jj) >> 1) - 1;   // 2^ctz(jj) - 1
            far_hi = (jj != 0 && w0 + d < n_valid) ? ipsi_hi_global(src[d], tabs) : 0ull;
        }
        __syncthreads();
        // ---- my 32 elements: limb -> planes, in place
        const uint32_t e0 = 32 * t;
#pragma unroll 1
        for (int L = 0; L < 4; L++) {
            uint32_t x[32];
#pragma unroll
            for (int j = 0; j < 32; j++) x[j] = S[L * IB_TILE + ib_swz(e0 + j)];
            transpose32(x);
#pragma unroll
            for (int j = 0; j < 32; j++) S[L * IB_TILE + ib_swz(e0 + j)] = x[j];
        }
        // ---- output limbs 2, 3 (hi64): planes -> elements, kept in H
        {
            uint32_t a2[32], a3[32], x[32];
#pragma unroll
            for (int j = 0; j < 32; j++) { a2[j] = 0; a3[j] = 0; }
#pragma unroll
            for (int L = 0; L < 4; L++) {
#pragma unroll
                for (int j = 0; j < 32; j++) x[j] = S[L * IB_TILE + ib_swz(e0 + j)];
                if (L == 0) { bs_ipsi_2_0(x, a2); bs_ipsi_3_0(x, a3); }
                else if (L == 1) { bs_ipsi_2_1(x, a2); bs_ipsi_3_1(x, a3); }
                else if (L == 2) { bs_ipsi_2_2(x, a2); bs_ipsi_3_2(x, a3); }
                else { bs_ipsi_2_3(x, a2); bs_ipsi_3_3(x, a3); }
            }
            transpose32(a2);
            transpose32(a3);
#pragma unroll
            for (int j = 0; j < 32; j++) { H[ib_swz(e0 + j)] = a2[j]; H[IB_TILE + ib_swz(e0 + j)] = a3[j]; }
        }
        // ---- output limbs 0, 1 (lo64)
        uint32_t a0[32], a1[32];
        {
            uint32_t x[32];
#pragma unroll
            for (int j = 0; j < 32; j++) { a0[j] = 0; a1[j] = 0; }
#pragma unroll
            for (int L = 0; L < 4; L++) {
#pragma unroll
                for (int j = 0; j < 32; j++) x[j] = S[L * IB_TILE + ib_swz(e0 + j)];
                if (L == 0) { bs_ipsi_0_0(x, a0); bs_ipsi_1_0(x, a1); }
                else if (L == 1) { bs_ipsi_0_1(x, a0); bs_ipsi_1_1(x, a1); }
                else if (L == 2) { bs_ipsi_0_2(x, a0); bs_ipsi_1_2(x, a1); }
                else { bs_ipsi_0_3(x, a0); bs_ipsi_1_3(x, a1); }
            }
            transpose32(a0);
            transpose32(a1);
        }
        __syncthreads();   // H complete; every thread done with the planes
        // ---- combine: out[w] = lo64(C_w) ^ hi64(C_(w-1)); staged limb-planar in S (limbs 0, 1)
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const uint32_t e = e0 + j;
            const uint64_t jj = (w0 + e) & (N - 1);
            uint32_t plo, phi;
            if (e == 0) { plo = (uint32_t)halo_hi; phi = (uint32_t)(halo_hi >> 32); }
            else if (jj == 0) { plo = 0; phi = 0; }   // first word of a product
            else { plo = H[ib_swz(e - 1)]; phi = H[IB_TILE + ib_swz(e - 1)]; }
            if (MC && jj != 0) {
                if (jj & 1) { plo ^= H[ib_swz(e)]; phi ^= H[IB_TILE + ib_swz(e)]; }
                else if (e == 0) { plo ^= (uint32_t)far_hi; phi ^= (uint32_t)(far_hi >> 32); }
                else {   // e != 0: ctz(jj) = ctz(e) < 12, the partner lies in this tile and product
                    const uint32_t q = ib_swz(e + (e & (0u - e)) - 1);
                    plo ^= H[q]; phi ^= H[IB_TILE + q];
                }
            }
            S[ib_swz(e)] = a0[j] ^ plo;
            S[IB_TILE + ib_swz(e)] = a1[j] ^ phi;
        }
        __syncthreads();
        uint64_t* dst = out + pair * N + w0;   // (pair = 0: flat)
        for (uint32_t e = t; e < IB_TILE; e += IB_THREADS) {
            const uint32_t q = ib_swz(e);
            if (w0 + e < n_write) dst[e] = ((uint64_t)S[IB_TILE + q] << 32) | S[q];
        }
        __syncthreads();
    }
}

// =============================================================================================
// Host side: tables, planning, workspace, entry points
// =============================================================================================
static thread_local std::string g_last_error;

// ------------------------------------------------------------------------------ profiling hook
struct ProfRec {
    std::string name;
    cudaEvent_t beg, end;
    double bytes;   // algorithmic HBM bytes of the launch
    double ops;     // algorithmic ALU-pipe lane instructions of the launch (ALU-bound designs), else 0
    int launches;   // kernel launches inside the bracket
};
// Designed ALU-pipe instructions (SASS, per lane) of the arithmetic cores, counted from cuobjdump:
//   one bit-sliced TGF(2^32) product (bs_mul32, 32 elements): 868 LOP3
//   one table butterfly of k_fft2 (4 limbs x (8 PRMT + 2 nibble masks + 2 shifts + 4 XOR3) + 4 XOR): 68
#define OPS_BS_MUL32 868.0
//   the same product by a multiplier below 2^16 / 2^8 (bs_mul_w: 2 x bs_mul16 / 4 x bs_mul8): 2 x 259 / 4 x 80 LOP3
#define OPS_BS_MUL16 518.0
#define OPS_BS_MUL8 320.0
// designed ALU-pipe instructions of one k_bottom launch: per 2^11-element tile, 2 (forward) + 1 (inverse) x 128
// products per layer at the layer's multiplier width, 576 general products of the pointmul
static double bottom_alu_ops(const BottomParams& bp) {
    double per_tile = (bp.mode & 2) ? 576.0 * OPS_BS_MUL32 : 0.0;
    const double nl = ((bp.mode & 1) ? 2.0 : 0.0) + ((bp.mode & 4) ? 1.0 : 0.0);
    for (int k = 0; k < bp.L; k++) {
        const int wc = bp.m + bp.map.bits - k;
        per_tile += nl * 128.0 * (wc <= 8 ? OPS_BS_MUL8 : (wc <= 16 ? OPS_BS_MUL16 : OPS_BS_MUL32));
    }
    return (double)bp.ntiles * per_tile;
}
#define OPS_M4R_BUTTERFLY 68.0
static thread_local bool g_prof_on = false;
static thread_local std::vector<ProfRec> g_prof;
static thread_local std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t prof_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
static void prof_clear() {
    for (auto& r : g_prof) {
        g_event_pool.push_back(r.beg);
        g_event_pool.push_back(r.end);
    }
    g_prof.clear();
}
// RAII bracket around one kernel launch
struct ProfScope {
    int idx = -1;
    cudaStream_t st;
    ProfScope(const char* name, double bytes, cudaStream_t s, double ops = 0.0, int launches = 1) : st(s) {
        if (!g_prof_on) return;
        ProfRec r{name, prof_event(), prof_event(), bytes, ops, launches};
        cudaEventRecord(r.beg, st);
        g_prof.push_back(r);
        idx = (int)g_prof.size() - 1;
    }
    ~ProfScope() {
        if (idx >= 0) cudaEventRecord(g_prof[idx].end, st);
    }
};

static bool env_flag(const char* name) {
    static std::mutex mu;
    static std::map<std::string, bool> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(name);
    if (it != cache.end()) return it->second;
    // unset, empty, "0", "false", "no" and "off" are false; anything else is true
    const char* e = getenv(name);
    bool v = e != nullptr && e[0] != 0;
    if (v) {
        std::string t(e);
        for (auto& ch : t) ch = (char)tolower((unsigned char)ch);
        v = !(t == "0" || t == "false" || t == "no" || t == "off");
    }
    cache[name] = v;
    return v;
}

// integer knob: the default unless the variable holds an integer in [lo, hi]
static int env_int(const char* name, int dflt, int lo, int hi) {
    const char* e = getenv(name);
    if (!e || !e[0]) return dflt;
    char* end = nullptr;
    const long v = strtol(e, &end, 10);
    return (end && *end == 0 && v >= lo && v <= hi) ? (int)v : dflt;
}
// per-call flag (not cached): unset, empty or "0" = off
static bool env_flag_now(const char* name) {
    const char* e = getenv(name);
    return e && e[0] && !(e[0] == '0' && e[1] == 0);
}

static gf2x_status fail(gf2x_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}
#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) return fail(GF2X_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

struct DeviceState {
    DevTables* tabs = nullptr;
    DevTables* host = nullptr;   // host copy (multiplier images for host-side constants)
    struct DevTables256* tabs256 = nullptr;   // w = 128 tables (w128.cuh), built on first use
    struct DevTablesA4* tabsA4 = nullptr;     // Alg. 4 tables (alg4.cuh), built on first use
    std::map<int, uint4*> frob;               // App. C constants per m (frob.cuh), built on first use
    std::map<int, uint32_t*> small_kt;        // k_small FFT constants per (m, segments) (get_small_kt)
    void* shard_ws = nullptr;    // simulation workspace (gf2x_mul_sharded_sim)
    size_t shard_ws_bytes = 0;
    int sm_count = 0;
    std::map<cudaStream_t, std::pair<void*, size_t>> ws;  // per-stream workspace cache (stream_workspace)
    std::vector<void*> retired;            // outgrown workspaces (a captured graph may still use them)
    struct Aux {
        cudaStream_t s = nullptr;          // side stream (high priority) for independent sub-chains
        cudaEvent_t fork = nullptr, join = nullptr;
    };
    std::map<cudaStream_t, Aux> aux;       // per caller stream
};
static std::mutex g_mu;
static std::map<int, DeviceState> g_dev;

static void host_build_tables(DevTables* T) {
    using namespace gf2x_host;
    memset(T, 0, sizeof(DevTables));
    Isomorphism iso = build_isomorphism();
    // psi64: chunk ch of a 64-bit polynomial-basis block
    for (int ch = 0; ch < 8; ch++)
        for (int x = 0; x < 256; x++) {
            u128 v = 0;
            for (int b = 0; b < 8; b++)
                if ((x >> b) & 1) v ^= iso.polyToTower[8 * ch + b];
            T->psi64[ch * 256 + x] = make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96));
        }
    for (int ch = 0; ch < 16; ch++)
        for (int x = 0; x < 256; x++) {
            u128 v = 0;
            for (int b = 0; b < 8; b++)
                if ((x >> b) & 1) v ^= iso.towerToPoly[8 * ch + b];
            T->ipsi[ch * 256 + x] = make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96));
        }
    // wt: c -> c * v_(4t) restricted to byte position pos of c
    for (int t = 1; t < 8; t++)
        for (int pos = 0; pos < 4; pos++)
            for (int x = 0; x < 256; x++) {
                u128 c = ((u128)x) << (8 * pos);
                T->wt[(t - 1) * 1024 + pos * 256 + x] = (uint32_t)mul_basis(c, 4 * t);
            }
    // S[k][j] = s_k(v_j), k, j < 32
    for (int j = 0; j < 32; j++) {
        u128 v = ((u128)1) << j;
        for (int k = 0; k < 32; k++) {
            T->S[k * 32 + j] = (uint32_t)v;
            v = s1(v);
        }
    }
}

static gf2x_status get_device(int* dev_out, DeviceState** st_out) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceState& st = g_dev[dev];
    if (!st.tabs) {
        DevTables* h = new DevTables;
        host_build_tables(h);
        DevTables* d = nullptr;
        cudaError_t e = cudaMalloc(&d, sizeof(DevTables));
        if (e != cudaSuccess) { delete h; return fail(GF2X_ENOMEM, "table allocation failed"); }
        e = cudaMemcpy(d, h, sizeof(DevTables), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_S, h->S, sizeof(h->S));
        if (e != cudaSuccess) { delete h; cudaFree(d); return fail(GF2X_ECUDA, cudaGetErrorString(e)); }
        st.host = h;
        CUDA_TRY(cudaDeviceGetAttribute(&st.sm_count, cudaDevAttrMultiProcessorCount, dev));
        // opt-in shared memory sizes
#define FFT_ATTR(a, b, c) CUDA_TRY(cudaFuncSetAttribute(k_fft2<a, b, c>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024))
        FFT_ATTR(false, false, false); FFT_ATTR(false, false, true); FFT_ATTR(false, true, false); FFT_ATTR(false, true, true);
        FFT_ATTR(true, false, false); FFT_ATTR(true, false, true);
#undef FFT_ATTR
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_tile<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_tile<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_bottom<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_bottom<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#define RB_ATTR(T, W) CUDA_TRY(cudaFuncSetAttribute(k_cvt_rb<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_rb_tma<uint64_t, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_rb_tma<uint4, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        RB_ATTR(uint64_t, 2); RB_ATTR(uint64_t, 3); RB_ATTR(uint64_t, 4); RB_ATTR(uint64_t, 5); RB_ATTR(uint64_t, 6);
        RB_ATTR(uint4, 2); RB_ATTR(uint4, 3); RB_ATTR(uint4, 4); RB_ATTR(uint4, 5); RB_ATTR(uint4, 6);
#undef RB_ATTR
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_res<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_res<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#define SEAM_ATTR(T, BH) CUDA_TRY(cudaFuncSetAttribute(k_cvt_seam<T, BH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        SEAM_ATTR(uint64_t, 1) SEAM_ATTR(uint64_t, 2) SEAM_ATTR(uint64_t, 3) SEAM_ATTR(uint64_t, 4)
        SEAM_ATTR(uint4, 1) SEAM_ATTR(uint4, 2) SEAM_ATTR(uint4, 3) SEAM_ATTR(uint4, 4)
#undef SEAM_ATTR
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_top<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_top<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_slab<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_small<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_small<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_small<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_small<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_small<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_slab<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_ipsi_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_ipsi_bs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_ipsi_bs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        st.tabs = d;
    }
    *dev_out = dev;
    *st_out = &st;
    return GF2X_OK;
}

// ------------------------------------------------------------------------------ planning
static int ceil_log2_u64(uint64_t x) {
    int r = 0;
    while ((1ull << r) < x) r++;
    return r;
}

// BasisCvt schedule (Alg. 3 with the paper's largest-K split, R4-R6) as global ops.
// The inner conversions (windows inside [sigma, sigma+K)) and the outer one (windows inside
// [sigma+K, sigma+m)) act on disjoint index bits, so they commute (R14); the inner ones
// are emitted first because their windows continue where the Taylor steps end.
static void cvt_ops(int m, int sigma, std::vector<CvtOp>& out) {
    if (m <= 1) return;
    int K = 1;
    while (2 * K <= m - 1) K *= 2;
    for (int l = m; l >= K + 1; --l) out.push_back({l + sigma, K});
    cvt_ops(K, sigma, out);
    cvt_ops(m - K, sigma + K, out);
}

struct CvtPass {
    bool stream;
    bool res = false;        // residue-class pass (k_cvt_res) over a run of same-K Taylor steps
    int c, r_lo, R;          // tile passes
    int q = 0, C_log = 0, rows = 0;   // residue passes: chunk bits, classes per tile, rows per class
    bool rb = false;         // register-blocked pass (k_cvt_rb): K <= 4 steps inside 8 index bits
    CvtRbParams rbp;         // its geometry, phases and op codes (data/sizes filled at launch)
    int rb_wb = 0;           // phase width (bits)
    std::vector<CvtOp> ops;  // tile / residue: ops in forward execution order; stream: 1 op
};

// Try to take a run of ops starting at ops[oi] as one register-blocked pass; returns the number taken.
static int plan_rb(const std::vector<CvtOp>& ops, size_t oi, int m, int unit_bytes, CvtPass& P) {
    int lo = 64, hi = 0;
    size_t e = oi;
    for (; e < ops.size() && (int)(e - oi) < RB_MAX_OPS; e++) {
        if (ops[e].K > 4) break;
        const int a = ops[e].lg - 1 - ops[e].K, b = ops[e].lg;
        const int nlo = std::min(lo, a), nhi = std::max(hi, b);
        if (nhi - nlo > 8) break;
        lo = nlo; hi = nhi;
    }
    if (e == oi) return 0;
    const int R = hi - lo;
    const int Cw = unit_bytes == 8 ? 4 : 3;   // 128-byte rows; 32 KB tiles (double-buffered: 3 CTAs/SM)
    int mode, C;
    if (lo == 0) { mode = 1; C = std::min(Cw, m - R); }
    else if (lo >= Cw) { mode = 0; C = Cw; }
    else return 0;
    const int WB = std::min(6, R);
    CvtRbParams& q = P.rbp;
    memset(&q, 0, sizeof(q));
    q.r_lo = lo; q.R = R; q.C = C; q.mode = mode;
    int nph = 0, plo = 64, phi = 0, cnt = 0;
    std::vector<std::pair<int, int>> win;   // op windows relative to lo
    for (size_t i = oi; i < e; i++) win.push_back({ops[i].lg - 1 - ops[i].K - lo, ops[i].lg - lo});
    size_t first = 0;
    auto flush = [&](size_t upto) {
        const int w_lo = std::min(plo, R - WB);
        q.ph_lo[nph] = w_lo;
        q.ph_n[nph] = (int)(upto - first);
        for (size_t i = first; i < upto; i++) {
            const int K = ops[oi + i].K;
            const int kk = K == 1 ? 0 : (K == 2 ? 1 : 2);
            q.ops[cnt++] = (unsigned char)(kk | ((win[i].first - w_lo) << 2));
        }
        nph++;
        first = upto;
    };
    for (size_t i = 0; i < win.size(); i++) {
        const int nlo = std::min(plo, win[i].first), nhi = std::max(phi, win[i].second);
        if (nhi - nlo > WB) {
            if (nph + 1 >= RB_MAX_PHASES) return 0;
            flush(i);
            plo = win[i].first; phi = win[i].second;
        } else {
            plo = nlo; phi = nhi;
        }
    }
    flush(win.size());
    q.nphase = nph;
    P.stream = false; P.res = false; P.rb = true; P.rb_wb = WB;
    P.c = P.r_lo = P.R = 0;
    P.ops.assign(ops.begin() + oi, ops.begin() + e);
    return (int)(e - oi);
}

// Greedy grouping of consecutive ops into tile passes: a pass holds tile bits [0,T) (contiguous)
// or [0,cmin) U [r_lo, r_lo + T - cmin) (rows of 2^cmin contiguous units = one 32-byte sector);
// an op whose window is wider than a tile streams through HBM.
static std::vector<CvtPass> plan_cvt_ops(const std::vector<CvtOp>& ops, int m, int unit_bytes);
static std::vector<CvtPass> plan_cvt(int m, int unit_bytes) {
    std::vector<CvtOp> ops;
    cvt_ops(m, 0, ops);
    return plan_cvt_ops(ops, m, unit_bytes);
}
// ops: in forward execution order, windows inside [0, m)
static std::vector<CvtPass> plan_cvt_ops(const std::vector<CvtOp>& ops, int m, int unit_bytes) {
    const int T = std::min(m, unit_bytes == 8 ? 14 : 13);  // 128 KB tiles
    const int cmin = unit_bytes == 8 ? 2 : 1;
    const int Rrow = T - cmin;
    std::vector<CvtPass> passes;
    int span_lo = 0, span_hi = 0;
    auto close = [&](CvtPass& P) {
        if (P.stream || P.res || P.rb) return;
        if (span_hi <= T) { P.c = 0; P.r_lo = 0; P.R = T; }
        else { P.c = cmin; P.R = Rrow; P.r_lo = std::max(cmin, std::min(span_lo, m - Rrow)); }
    };
    auto fits = [&](int lo, int hi) { return hi <= T || (lo >= cmin && hi - lo <= Rrow); };
    for (size_t oi = 0; oi < ops.size(); oi++) {
        const CvtOp& op = ops[oi];
        const int wlo = op.lg - 1 - op.K, whi = op.lg;
        // K=8 runs also as residue passes (measured faster than 2 tile passes); a lone K=8 step that fits a tile
        // (the top step of a 2^9-unit product) stays in the tile passes
        bool res8 = op.K == 8 && !env_flag("GF2X_NO_RES8");
        if (res8 && fits(wlo, whi) && !(oi + 1 < ops.size() && ops[oi + 1].K == 8 && ops[oi + 1].lg == op.lg - 1) &&
            !env_flag("GF2X_RES8_SINGLE"))
            res8 = false;
        if ((!fits(wlo, whi) || res8) && op.lg <= 31) {
            // a run of same-K steps at descending levels whose windows exceed a tile: one
            // residue-class pass if the rows of a class fit shared memory (else this step streams)
            size_t e = oi + 1;
            while (e < ops.size() && ops[e].K == op.K && ops[e].lg == ops[e - 1].lg - 1 &&
                   (res8 || !fits(ops[e].lg - 1 - ops[e].K, ops[e].lg)))
                e++;
            const uint64_t M = (1ull << op.K) - 1;
            const int rows = (int)(((1ull << op.lg) - 1) / M + 1);
            int C_log = unit_bytes == 8 ? 4 : 3;   // >= 128-byte runs per row
            const size_t budget = 33 * 1024;       // per buffer (k_cvt_res is double-buffered, 3 CTAs/SM)
            if ((size_t)rows * ((size_t)1 << C_log) * unit_bytes <= budget) {
                while (C_log < 6 && (size_t)rows * ((size_t)2 << C_log) * unit_bytes <= budget) C_log++;
                // the kernel keeps RES_MAXJ row slots per thread (RES_THREADS / 2^C_log row lanes)
                const int maxj = unit_bytes == 8 ? RES_MAXJ : RES_SLOTS128;
                while (C_log > 0 && rows > maxj * (RES_THREADS >> C_log)) C_log--;
                if (!passes.empty()) close(passes.back());
                CvtPass P;
                P.stream = false;
                P.res = true;
                P.c = P.r_lo = P.R = 0;
                P.q = op.lg;
                P.C_log = C_log;
                P.rows = rows;
                P.ops.assign(ops.begin() + oi, ops.begin() + e);
                passes.push_back(P);
                span_lo = 0; span_hi = 64;   // nothing joins a residue pass
                oi = e - 1;
                continue;
            }
        }
        if (!env_flag("GF2X_NO_RB")) {
            CvtPass P;
            const int took = plan_rb(ops, oi, m, unit_bytes, P);
            if (took > 0) {
                if (!passes.empty()) close(passes.back());
                passes.push_back(P);
                span_lo = 0; span_hi = 64;
                oi += took - 1;
                continue;
            }
        }
        if (!passes.empty() && !passes.back().stream && !passes.back().res && !passes.back().rb &&
            (int)passes.back().ops.size() < MAX_TILE_OPS) {
            const int nlo = std::min(span_lo, wlo), nhi = std::max(span_hi, whi);
            if (fits(nlo, nhi)) {
                passes.back().ops.push_back(op);
                span_lo = nlo; span_hi = nhi;
                continue;
            }
        }
        if (!passes.empty()) close(passes.back());
        CvtPass P;
        P.stream = !fits(wlo, whi);
        P.c = P.r_lo = P.R = 0;
        P.ops.push_back(op);
        passes.push_back(P);
        span_lo = wlo; span_hi = whi;
    }
    if (!passes.empty()) close(passes.back());
    return passes;
}

struct FftPass {
    int c, k_lo, k_hi;  // direct: tile bits [0,c) U [k_lo,k_hi); bottom: c = k_lo = 0, k_hi = Rt
    bool bottom;
    int layers;         // bottom: layers [0, layers)
};
// forward order (top-down); the first pass also applies changeRepr.  The high layers [bot, m) go to
// table passes of <= 6 layers for the changeRepr pass (its 32 KB psi table) and <= 7 below it (127 M4R
// tables, 64 KB; their tables are rebuilt only when the tile's bits >= k_hi change); layers
// [0, min(m, bot)) form the bit-sliced bottom pass: 6 layers (5 measured 0.5 % slower at c4b, 8 % at c3),
// except for short transforms (m <= 10: one table pass either way; 5 measured 10 % faster at c2).
static int fft_passes(int H, int maxr) { return H <= 0 ? 0 : (H <= 6 ? 1 : 1 + (H - 6 + maxr - 1) / maxr); }
static std::vector<FftPass> plan_fft(int m) {
    static const int maxr = env_int("GF2X_MAXR", 7, 1, 7);
    static const int forced = env_int("GF2X_BOT_B", 0, 1, BOT_B_MAX);
    const int bot = forced ? forced : (m <= 10 ? 5 : 6);
    std::vector<FftPass> v;
    const int H = m > bot ? m - bot : 0;
    const int np = fft_passes(H, maxr);
    int top = m;
    for (int i = 0; i < np; i++) {
        const int rem = top - bot;
        const int r = i == 0 ? std::min(6, rem - (np - 1)) : (rem + (np - i) - 1) / (np - i);
        const int lo = top - r;
        // 32-column tiles (2 CTAs/SM) for the changeRepr pass and passes of >= 6 layers; 64 columns (one
        // double-buffered CTA per SM) for shorter passes (measured: c4b -1.7 %, c4a / c5 -0.3 % vs 64 columns
        // for 6-layer passes)
        static const int cdir = env_int("GF2X_FFT_C", 6, 5, 6);
        int c = (i == 0 || r >= 6) ? 5 : cdir;
        if (c > lo) c = lo;   // column bits must lie below the pass's layers
        v.push_back({c, lo, top, false, 0});
        top = lo;
    }
    v.push_back({0, 0, 0, true, m < bot ? m : bot});  // the fused bit-sliced bottom kernel
    return v;
}

// A conversion of n units in a 2^(p+1) array, n <= 2^p + 2^j, done as a 2^p conversion of the lower
// half plus a 2^j conversion of the tail and the s_p(x) = sum_{q subset p} x^(2^q) shifts (R22)
struct CvtSplit {
    int p = -1, j = 0;
    std::vector<CvtPass> lo, hi;
};
static CvtSplit plan_cvt_split(uint64_t n, int mfull, int unit_bytes) {
    CvtSplit S;
    if (env_flag("GF2X_NO_CVT_SPLIT") || mfull < 16) return S;
    const int p = mfull - 1;
    if (n <= (1ull << p)) return S;
    const int j = ceil_log2_u64(n - (1ull << p));
    if (j > p - 2) return S;   // a tail above a quarter saves too little
    S.p = p; S.j = j;
    S.lo = plan_cvt(p, unit_bytes);
    S.hi = plan_cvt(j, unit_bytes);
    return S;
}
static int lucas_shifts(int p, uint64_t* off) {   // 2^q for q subset of p, q != p (the lower terms of s_p)
    int n = 0;
    for (int q = 0; q < p; q++)
        if ((q & p) == q) off[n++] = 1ull << q;
    return n;
}

struct Plan {
    uint64_t na, nb, N, batch;
    uint64_t a_bits = 0, b_bits = 0;
    int m, ma, mb;
    std::vector<CvtPass> cvt_a, cvt_b, icvt;
    std::vector<CvtPass> icvt64;   // R28: iBasisCvt of the combined 64-bit sequence (mcomb_ok)
    std::vector<FftPass> fft;
    size_t off_sa, off_sb, off_wa, off_wb, bytes;
    // one product: BasisCvt split at 2^p + tail 2^j (R22); p < 0 = not split
    CvtSplit sa, sb, ic;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static void dump_plan(const Plan& P) {
    auto dc = [](const char* nm, const std::vector<CvtPass>& v) {
        fprintf(stderr, "[gf2x plan] %s:", nm);
        for (auto& p : v) {
            if (p.stream) fprintf(stderr, " stream(%d,%d)", p.ops[0].lg - 1 - p.ops[0].K, p.ops[0].lg);
            else if (p.res) fprintf(stderr, " res{q=%d K=%d lg=%d..%d C=%d rows=%d}", p.q, p.ops[0].K, p.ops[0].lg,
                                    p.ops.back().lg, 1 << p.C_log, p.rows);
            else if (p.rb) fprintf(stderr, " rb{rows=[%d,%d) C=%d mode=%d phases=%d ops=%zu}", p.rbp.r_lo, p.rbp.r_lo + p.rbp.R,
                                   p.rbp.C, p.rbp.mode, p.rbp.nphase, p.ops.size());
            else fprintf(stderr, " tile{c=%d rows=[%d,%d) ops=%zu}", p.c, p.r_lo, p.r_lo + p.R, p.ops.size());
        }
        fprintf(stderr, "\n");
    };
    dc("cvt_a", P.cvt_a);
    dc("icvt", P.icvt);
    fprintf(stderr, "[gf2x plan] fft:");
    for (auto& f : P.fft) {
        if (f.bottom) fprintf(stderr, " bottom{layers=%d}", f.layers);
        else fprintf(stderr, " direct{c=%d [%d,%d)}", f.c, f.k_lo, f.k_hi);
    }
    fprintf(stderr, "\n");
}

static gf2x_status make_plan(uint64_t a_bits, uint64_t b_bits, int64_t batch, Plan& P) {
    if (batch < 0) return fail(GF2X_EINVAL, "negative batch");
    P.na = (a_bits + 63) / 64;
    P.nb = (b_bits + 63) / 64;
    P.a_bits = a_bits;
    P.b_bits = b_bits;
    P.batch = (uint64_t)batch;
    const uint64_t L = P.na + P.nb - 1;
    P.m = ceil_log2_u64(L);
    if (P.m > 32) return fail(GF2X_ETOOBIG, "FFT size exceeds 2^32 points");
    P.N = 1ull << P.m;
    P.ma = ceil_log2_u64(P.na);
    P.mb = ceil_log2_u64(P.nb);
    P.cvt_a = plan_cvt(P.ma, 8);
    P.cvt_b = plan_cvt(P.mb, 8);
    P.icvt = plan_cvt(P.m, 16);
    P.icvt64 = plan_cvt(P.m, 8);
    P.fft = plan_fft(P.m);
    if (P.batch == 1) {
        P.sa = plan_cvt_split(P.na, P.ma, 8);
        P.sb = plan_cvt_split(P.nb, P.mb, 8);
        P.ic = plan_cvt_split(L, P.m, 16);
    }
    // workspace: Sa | Sb (u64 blocks) and Wa | Wb (spectra) each contiguous, so that passes with
    // equal shapes for a and b run as one launch over 2*batch products; a 2^11-element pad after Wb
    // keeps the bottom kernel's last tile in bounds
    P.off_sa = 0;
    P.off_sb = (P.off_sa + (1ull << P.ma) * P.batch * 8 + 15) & ~(size_t)15;   // 16-byte aligned (vector / bulk access)
    P.off_wa = align256(P.off_sb + (1ull << P.mb) * P.batch * 8);
    P.off_wb = P.off_wa + P.N * P.batch * 16;
    P.bytes = align256(P.off_wb + (P.N * P.batch + 2048) * 16);
    if (env_flag("GF2X_DEBUG_PLAN")) dump_plan(P);
    return GF2X_OK;
}

static bool slab_triple(const std::vector<CvtPass>& v, size_t i, int m);
// launches of a planned conversion (a CVT(16) slab triple is one launch)
static int cvt_launches(const std::vector<CvtPass>& v, int m) {
    int n = 0;
    for (size_t i = 0; i < v.size(); i++, n++)
        if (slab_triple(v, i, m)) i += 2;
    return n;
}
static int launches_of_split(const CvtSplit& S, const std::vector<CvtPass>& full, int mfull) {
    return S.p < 0 ? cvt_launches(full, mfull) : 1 + cvt_launches(S.lo, S.p) + cvt_launches(S.hi, S.j);
}
static int top_rowbits(const CvtPass& p, int m);
// Split fused into the first forward conversion pass: a and b convert in one launch (equal shapes, contiguous
// scratch) and that pass is a k_cvt_top pass
static bool split_fused(const Plan& P) {
    const bool same = P.ma == P.mb && P.off_sb == P.off_sa + (1ull << P.ma) * P.batch * 8 && P.sa.p < 0 && P.sb.p < 0;
    return same && P.a_bits == P.b_bits && !P.cvt_a.empty() && top_rowbits(P.cvt_a[0], P.ma) >= 0 && !env_flag("GF2X_NO_FUSED_SPLIT");
}
// R28: InterleavedCombine before iBasisCvt (k_ipsi_bs<true>, then iBasisCvt of 64-bit words in the output
// buffer): the output holds all N words of every product (n_out = N), no split conversion, whole ipsi tiles
static bool mcomb_ok(const Plan& P) {
    return P.na + P.nb == P.N && P.ic.p < 0 && (P.N * P.batch) % IB_TILE == 0 && !env_flag("GF2X_NO_MCOMB") &&
           !env_flag("GF2X_NO_IPSI_BS");
}
static int small_cluster(const Plan& P);
static int launches_of(const Plan& P) {
    if (small_cluster(P)) return 1;
    const bool same = P.ma == P.mb && P.off_sb == P.off_sa + (1ull << P.ma) * P.batch * 8 && P.sa.p < 0 && P.sb.p < 0;
    int n = split_fused(P) ? 0 : 2;  // prep a, b
    n += launches_of_split(P.sa, P.cvt_a, P.ma) + (same ? 0 : launches_of_split(P.sb, P.cvt_b, P.mb)) +
         (mcomb_ok(P) ? cvt_launches(P.icvt64, P.m) : launches_of_split(P.ic, P.icvt, P.m));
    const int nd = (int)P.fft.size() - 1;
    n += (same ? 1 : 2) * (nd ? nd : 1);      // forward a, b (or the changeRepr-only pass)
    n += 1;                      // fused bottom
    n += nd;                     // inverse
    n += 1;                      // ipsi + combine
    return n;
}

// ------------------------------------------------------------------------------ launchers
static int grid_for(uint64_t items, int per_block, int sm_count, int occ) {
    uint64_t g = (items + per_block - 1) / per_block;
    uint64_t cap = (uint64_t)sm_count * occ;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// A residue pass that is the whole Taylor run of the top node with K = 16 over one chunk per pair (levels
// m .. 17) runs as k_cvt_top (generic classes as the superset-sum transform) when its rows fit a tile
static int top_rowbits(const CvtPass& p, int m) {
    if (!p.res || p.ops.empty() || env_flag("GF2X_NO_CVT_TOP")) return -1;
    const int K = p.ops[0].K;
    if (K != 16 || p.q != m || p.ops.front().lg != m || p.ops.back().lg != K + 1) return -1;
    if ((int)p.ops.size() != m - K) return -1;
    const int B = m - K;
    return (B >= 1 && B <= 9) ? B : -1;
}
// Split fused into the first forward conversion pass (k_cvt_top reads the caller's operands)
struct CvtSrc {
    const uint64_t* a;
    const uint64_t* b;
    uint64_t batch0, n, bits;
};

template <typename T>
static gf2x_status launch_cvt_top(const CvtPass& p, int B, T* data, int m, uint64_t batch, bool inverse, int sm_count,
                                  cudaStream_t st, const CvtSrc* src) {
    CvtTopParams prm;
    memset(&prm, 0, sizeof(prm));
    prm.data = data;
    prm.units_per_pair = 1ull << m;
    prm.batch = batch;
    prm.q = m; prm.K = 16; prm.B = B; prm.inverse = inverse ? 1 : 0;
    const size_t row_bytes = (((size_t)1 << B) + 1) * sizeof(T);   // one class, all rows
    int C_log = 0;
    while (C_log < 5 && row_bytes * ((size_t)2 << C_log) <= 33 * 1024) C_log++;
    prm.C_log = C_log;
    prm.c_gen = (1u << B) - 1 + (1u << (B - 1));
    if (src) {
        prm.src0 = src->a; prm.src1 = src->b; prm.batch0 = src->batch0; prm.nsrc = src->n; prm.bits = src->bits;
    }
    const size_t bufsz = ((row_bytes << C_log) + 127) & ~(size_t)127;
    const size_t sm = 2 * bufsz;
    const uint64_t M = (1ull << 16) - 1;
    const uint64_t ntiles = batch * ((M + (1ull << C_log) - 1) >> C_log);
    const int occ = std::max(1, std::min(3, (int)(200 * 1024 / (sm + 1024))));
    ProfScope ps(sizeof(T) == 8 ? "k_cvt_top<u64>" : "k_cvt_top<u128>",
                 (src ? 1.0 : 2.0) * (double)(1ull << m) * batch * sizeof(T) + (src ? (double)src->n * batch * 8 : 0.0), st);
    k_cvt_top<T><<<grid_for(ntiles, 1, sm_count, occ), TOP_THREADS, sm, st>>>(prm);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GF2X_OK : fail(GF2X_ECUDA, std::string("cvt top launch: ") + cudaGetErrorString(e));
}

// The passes i, i+1, i+2 of a plan are one CVT(16) node on 2^16-unit slabs (its K = 8 residue run, CVT(8) on
// bits [0, 8), CVT(8) on [8, 16)): they run as one k_cvt_slab launch
static bool slab_triple(const std::vector<CvtPass>& v, size_t i, int m) {
    if (i + 2 >= v.size() || m < SLAB_BITS || !env_flag("GF2X_CVT_SLAB")) return false;
    const CvtPass &a = v[i], &b = v[i + 1], &c = v[i + 2];
    if (!a.res || a.ops[0].K != 8 || a.q != 16 || a.ops.front().lg != 16 || a.ops.back().lg != 9 || a.ops.size() != 8)
        return false;
    if (!b.rb || b.rbp.r_lo != 0 || b.rbp.R != 8 || b.rbp.mode != 1 || b.rb_wb != 6) return false;
    if (!c.rb || c.rbp.r_lo != 8 || c.rbp.R != 8 || c.rbp.mode != 0 || c.rb_wb != 6) return false;
    return true;
}
// a residue pass that is a complete Taylor run (levels q .. K+1) with 5 <= B = q - K <= 8 row bits runs in
// the closed form of R27 (k_cvt_seam)
static bool seam_ok(const CvtPass& p) {
    if (!p.res || p.ops.empty() || env_flag("GF2X_NO_SEAM")) return false;
    const int K = p.ops[0].K, B = p.q - K;
    return B >= 5 && B <= 8 && p.ops.front().lg == p.q && (int)p.ops.size() == B && p.ops.back().lg == K + 1;
}
static CvtResParams res_params(const CvtPass& p, void* data, uint64_t per, uint64_t batch, bool inverse) {
    CvtResParams prm;
    prm.data = data;
    prm.units_per_pair = per;
    prm.batch = batch;
    prm.q = p.q;
    prm.K = p.ops[0].K;
    prm.lg_hi = p.ops.front().lg;
    prm.lg_lo = p.ops.back().lg;
    prm.inverse = inverse ? 1 : 0;
    prm.C_log = p.C_log;
    prm.rows = p.rows;
    return prm;
}
static size_t res_smem(const CvtPass& p, size_t unit) { return 2 * ((((size_t)p.rows << p.C_log) * unit + 127) & ~(size_t)127); }
static size_t rb_smem(const CvtRbParams& q, size_t unit) {
    const size_t ncols = (size_t)1 << q.C, nrows = (size_t)1 << q.R;
    return 2 * ((ncols * (nrows + (q.mode ? 16 / unit : 0)) * unit + 127) & ~(size_t)127);
}

template <typename T>
static gf2x_status launch_cvt_slab(const std::vector<CvtPass>& v, size_t i, T* data, int m, uint64_t batch, bool inverse,
                                   int sm_count, cudaStream_t st) {
    CvtSlabParams P;
    memset(&P, 0, sizeof(P));
    P.data = data;
    P.nslabs = (1ull << (m - SLAB_BITS)) * batch;
    P.inverse = inverse ? 1 : 0;
    P.res = res_params(v[i], data, 1ull << SLAB_BITS, 1, inverse);
    P.rb_lo = v[i + 1].rbp;
    P.rb_hi = v[i + 2].rbp;
    for (CvtRbParams* q : {&P.rb_lo, &P.rb_hi}) {
        q->units_per_pair = 1ull << SLAB_BITS;
        q->batch = 1;
        q->inverse = inverse ? 1 : 0;
    }
    const size_t sm = std::max(res_smem(v[i], sizeof(T)), std::max(rb_smem(P.rb_lo, sizeof(T)), rb_smem(P.rb_hi, sizeof(T))));
    static const int CS = env_int("GF2X_SLAB_CLUSTER", 8, 2, 8);
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(SLAB_THREADS);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    // as many clusters as can be resident at once (a persistent loop over the slabs)
    static int max_cl[2] = {0, 0};
    int& mc = max_cl[sizeof(T) == 8 ? 0 : 1];
    if (!mc) {
        cfg.gridDim = dim3(CS * (sm_count / CS));
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_cvt_slab<T>, &cfg) != cudaSuccess || n < 1) {
            cudaGetLastError();
            n = sm_count / CS;
        }
        mc = n;
    }
    const uint64_t ncl = std::min<uint64_t>(P.nslabs, (uint64_t)mc);
    cfg.gridDim = dim3((unsigned)(ncl * CS));
    ProfScope ps(sizeof(T) == 8 ? "k_cvt_slab<u64>" : "k_cvt_slab<u128>", 2.0 * (double)(1ull << m) * batch * sizeof(T), st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cvt_slab<T>, P);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? GF2X_OK : fail(GF2X_ECUDA, std::string("cvt slab launch: ") + cudaGetErrorString(e));
}

// ------------------------------------------------------------------------------ TMA tensor maps (k_cvt_rb_tma)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        else
            cudaGetLastError();
    }
    return fn;
}
// L2 prefetch of the next tile (GF2X_L2PF bit 0: k_bottom, bit 1: k_ipsi_bs on the R28 path)
static int bottom_l2pf() { static const int v = env_int("GF2X_L2PF", 1, 0, 3); return v & 1; }   // c4b: 1.941 -> 1.927 ms
static int ipsi_l2pf() { static const int v = env_int("GF2X_L2PF", 1, 0, 3); return (v >> 1) & 1; }   // (no change measured)
static bool rb_tma_enabled() { return !env_flag("GF2X_NO_RB_TMA"); }   // measured 5 % faster (c4b)
// mode 0: dims (column run of 2^C units, middle bits [C, r_lo), rows [r_lo, r_lo + R), the rest incl. pairs),
// box (2^C units, 1, 2^R, 1); units as 64-bit elements (u128: 2 per unit).  Mode 1 uses 1-D bulk copies.
template <typename T>
static bool make_rb_tmap(const CvtRbParams& q, CUtensorMap* tm) {
    memset(tm, 0, sizeof(*tm));
    if (q.mode) return true;
    auto fn = tmap_encode_fn();
    if (!fn) return false;
    const uint64_t EU = sizeof(T) / 8;
    const uint64_t total = q.units_per_pair * q.batch;
    cuuint64_t dims[4] = {((cuuint64_t)1 << q.C) * EU, (cuuint64_t)1 << (q.r_lo - q.C), (cuuint64_t)1 << q.R,
                          (cuuint64_t)(total >> (q.r_lo + q.R))};
    cuuint64_t strides[3] = {((cuuint64_t)1 << q.C) * sizeof(T), ((cuuint64_t)1 << q.r_lo) * sizeof(T),
                             ((cuuint64_t)1 << (q.r_lo + q.R)) * sizeof(T)};
    cuuint32_t box[4] = {(cuuint32_t)(((cuuint64_t)1 << q.C) * EU), 1, (cuuint32_t)1 << q.R, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (box[0] > 256 || box[2] > 256) return false;
    CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, q.data, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <typename T>
static gf2x_status run_cvt(const std::vector<CvtPass>& passes, T* data, int m, uint64_t batch, bool inverse,
                           int sm_count, cudaStream_t st, const CvtSrc* src = nullptr) {
    const uint64_t per = 1ull << m;
    std::vector<const CvtPass*> order;
    for (auto& p : passes) order.push_back(&p);
    if (inverse) std::reverse(order.begin(), order.end());
    for (size_t oi = 0; oi < order.size(); oi++) {
        // three passes forming a CVT(16) node on slabs: one cluster launch (in plan order i .. i+2)
        {
            const size_t pi = inverse ? passes.size() - 1 - oi : oi;   // plan index of this pass
            const size_t first = inverse ? (pi >= 2 ? pi - 2 : passes.size()) : pi;
            if (first < passes.size() && slab_triple(passes, first, m) && !(src && oi == 0)) {
                gf2x_status s = launch_cvt_slab<T>(passes, first, data, m, batch, inverse, sm_count, st);
                if (s != GF2X_OK) return s;
                oi += 2;
                continue;
            }
        }
        const CvtPass& p = *order[oi];
        const int topB = top_rowbits(p, m);
        if (src && oi == 0 && (topB < 0 || inverse || sizeof(T) != 8))
            return fail(GF2X_EINVAL, "fused Split needs a top Taylor pass first");
        // a top run with 5..8 row bits and no fused Split: the seam form covers every class (k_cvt_top runs Alg. 2's
        // sweeps on the first ~1.5 2^B classes)
        const bool top_seam = topB >= 0 && !(src && oi == 0) && seam_ok(p) && env_flag("GF2X_TOP_SEAM");
        if (topB >= 0 && !top_seam) {
            gf2x_status s = launch_cvt_top<T>(p, topB, data, m, batch, inverse, sm_count, st, oi == 0 ? src : nullptr);
            if (s != GF2X_OK) return s;
            continue;
        }
        if (p.rb) {
            CvtRbParams prm = p.rbp;
            prm.data = data;
            prm.units_per_pair = per;
            prm.batch = batch;
#ifdef GF2X_RB_NOPHASE_BUILD
            // measurement-only variant (build_variant with -DGF2X_RB_NOPHASE_BUILD): copy without converting
            prm.inverse = (inverse ? 1 : 0) | 2;
#else
            prm.inverse = inverse ? 1 : 0;
#endif
            // a node spanning all index bits of a (small) product: the tile's columns continue into the next
            // products (they are contiguous), up to the width the planner wanted
            if (prm.mode == 1 && prm.R + prm.C == m) {
                const int want = sizeof(T) == 8 ? 4 : 3;
                while (prm.C < want && (prm.batch & 1) == 0 && prm.batch > 1) {
                    prm.C++;
                    prm.units_per_pair <<= 1;
                    prm.batch >>= 1;
                }
            }
            const size_t ncols = (size_t)1 << prm.C, nrows = (size_t)1 << prm.R;
            const size_t bufsz = (ncols * (nrows + (prm.mode ? 16 / sizeof(T) : 0)) * sizeof(T) + 127) & ~(size_t)127;
            const size_t sm = 2 * bufsz;   // double-buffered
            const uint64_t ntiles = (prm.units_per_pair >> (prm.R + prm.C)) * prm.batch;
            const int occ = 3;
            ProfScope ps(sizeof(T) == 8 ? "k_cvt_rb<u64>" : "k_cvt_rb<u128>", 2.0 * per * batch * sizeof(T), st);
            const int g = grid_for(ntiles, 1, sm_count, occ);
            CUtensorMap tm;
            if (rb_tma_enabled() && p.rb_wb == 6 && make_rb_tmap<T>(prm, &tm)) {
                static const int st_tma = env_int("GF2X_RB_ST", 2, 0, 2);   // measured: 0.074 -> 0.068 ms per c4b pass
                prm.st_tma = st_tma;
                k_cvt_rb_tma<T, 6><<<g, RB_THREADS, sm, st>>>(prm, tm);
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("cvt rb tma launch: ") + cudaGetErrorString(e));
                continue;
            }
            switch (p.rb_wb) {
                case 2: k_cvt_rb<T, 2><<<g, RB_THREADS, sm, st>>>(prm); break;
                case 3: k_cvt_rb<T, 3><<<g, RB_THREADS, sm, st>>>(prm); break;
                case 4: k_cvt_rb<T, 4><<<g, RB_THREADS, sm, st>>>(prm); break;
                case 5: k_cvt_rb<T, 5><<<g, RB_THREADS, sm, st>>>(prm); break;
                default: k_cvt_rb<T, 6><<<g, RB_THREADS, sm, st>>>(prm); break;
            }
        } else if (p.res && seam_ok(p)) {
            const CvtResParams prm = res_params(p, data, per, batch, inverse);
            const uint64_t M = (1ull << prm.K) - 1, C = 32 / (sizeof(T) / 4);
            const uint64_t ntiles = (per >> p.q) * batch * ((M + C - 1) / C);
            ProfScope ps(sizeof(T) == 8 ? "k_cvt_seam<u64>" : "k_cvt_seam<u128>", 2.0 * per * batch * sizeof(T), st);
            const int g = grid_for(ntiles, 1, sm_count, 2);
            switch (p.q - prm.K) {
                case 5: k_cvt_seam<T, 1><<<g, SEAM_THREADS, seam_smem(), st>>>(prm); break;
                case 6: k_cvt_seam<T, 2><<<g, SEAM_THREADS, seam_smem(), st>>>(prm); break;
                case 7: k_cvt_seam<T, 3><<<g, SEAM_THREADS, seam_smem(), st>>>(prm); break;
                default: k_cvt_seam<T, 4><<<g, SEAM_THREADS, seam_smem(), st>>>(prm); break;
            }
        } else if (p.res) {
            CvtResParams prm;
            prm.data = data;
            prm.units_per_pair = per;
            prm.batch = batch;
            prm.q = p.q;
            prm.K = p.ops[0].K;
            prm.lg_hi = p.ops.front().lg;
            prm.lg_lo = p.ops.back().lg;
            prm.inverse = inverse ? 1 : 0;
            prm.C_log = p.C_log;
            prm.rows = p.rows;
            const size_t sm = 2 * ((((size_t)p.rows << p.C_log) * sizeof(T) + 127) & ~(size_t)127);
            const uint64_t M = (1ull << prm.K) - 1;
            const uint64_t ntiles = (per >> p.q) * batch * ((M + (1ull << p.C_log) - 1) >> p.C_log);
            const int occ = std::max(1, (int)(200 * 1024 / (sm + 1024)));
            ProfScope ps(sizeof(T) == 8 ? "k_cvt_res<u64>" : "k_cvt_res<u128>", 2.0 * per * batch * sizeof(T), st);
            k_cvt_res<T><<<grid_for(ntiles, 1, sm_count, std::min(occ, 3)), RES_THREADS, sm, st>>>(prm);
        } else if (p.stream) {
            const CvtOp op = p.ops[0];
            const uint64_t n = per * batch / 2;
            ProfScope ps(sizeof(T) == 8 ? "k_cvt_stream<u64>" : "k_cvt_stream<u128>", 3.0 * n * sizeof(T), st);
            k_cvt_stream<T><<<grid_for(n, 256, sm_count, 8), 256, 0, st>>>(data, per * batch, op.lg, op.K, inverse ? 1 : 0);
        } else {
            CvtTileParams prm;
            prm.data = data;
            prm.units_per_pair = per;
            prm.batch = batch;
            prm.c = p.c; prm.r_lo = p.r_lo; prm.R = p.R;
            prm.inverse = inverse ? 1 : 0;
            prm.nops = (int)p.ops.size();
            for (int i = 0; i < prm.nops; i++) prm.ops[i] = inverse ? p.ops[prm.nops - 1 - i] : p.ops[i];
            const size_t sm = ((size_t)1 << (p.c + p.R)) * sizeof(T);
            const uint64_t ntiles = (per >> (p.c + p.R)) * batch;
            ProfScope ps(sizeof(T) == 8 ? "k_cvt_tile<u64>" : "k_cvt_tile<u128>", 2.0 * per * batch * sizeof(T), st);
            k_cvt_tile<T><<<grid_for(ntiles, 1, sm_count, sm > 114 * 1024 ? 1 : 2), 512, sm, st>>>(prm);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("cvt launch: ") + cudaGetErrorString(e));
    }
    return GF2X_OK;
}

// R22 shifts: data[off_k + i] ^= data[src + i], i < n, for each offset (targets lie below src, so the
// source is read unchanged; targets of different offsets may coincide, hence the atomics)
struct ShiftList {
    uint64_t off[32];
    int n;
};
__device__ __forceinline__ void atomic_xor_unit(uint64_t* p, uint64_t v) { atomicXor((unsigned long long*)p, (unsigned long long)v); }
__device__ __forceinline__ void atomic_xor_unit(uint4* p, uint4 v) {
    unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
    const unsigned long long lo = ((unsigned long long)v.y << 32) | v.x, hi = ((unsigned long long)v.w << 32) | v.z;
    if (lo) atomicXor(q, lo);
    if (hi) atomicXor(q + 1, hi);
}
__device__ __forceinline__ bool unit_nonzero(uint64_t v) { return v != 0; }
__device__ __forceinline__ bool unit_nonzero(uint4 v) { return (v.x | v.y | v.z | v.w) != 0; }
template <typename T>
__global__ void __launch_bounds__(256) k_shift_xor(T* __restrict__ data, uint64_t src, uint64_t n, ShiftList sl) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const T v = data[src + i];
        if (!unit_nonzero(v)) continue;
        for (int k = 0; k < sl.n; k++) atomic_xor_unit(data + sl.off[k] + i, v);
    }
}
template <typename T>
static gf2x_status launch_shift_xor(T* data, int p, uint64_t n, int smc, cudaStream_t st) {
    ShiftList sl;
    sl.n = lucas_shifts(p, sl.off);
    ProfScope ps("k_shift_xor", (double)n * sizeof(T) * (1 + 2 * sl.n), st);
    k_shift_xor<T><<<grid_for(n, 256, smc, 8), 256, 0, st>>>(data, 1ull << p, n, sl);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GF2X_OK : fail(GF2X_ECUDA, std::string("shift launch: ") + cudaGetErrorString(e));
}
// forward BasisCvt of one operand (n units, zero beyond) per R22: f_lo += sum_{q subset p, q != p} x^(2^q) f_hi,
// then BasisCvt_p(f_lo) and BasisCvt_j(f_hi) in place
static gf2x_status run_cvt_fwd_split(const CvtSplit& S, uint64_t* data, uint64_t n, int smc, cudaStream_t st) {
    gf2x_status s;
    if ((s = launch_shift_xor<uint64_t>(data, S.p, n - (1ull << S.p), smc, st)) != GF2X_OK) return s;
    if ((s = run_cvt<uint64_t>(S.lo, data, S.p, 1, false, smc, st)) != GF2X_OK) return s;
    return run_cvt<uint64_t>(S.hi, data + (1ull << S.p), S.j, 1, false, smc, st);
}
// inverse per R22: iBasisCvt_p(g_lo) + s_p(x) iBasisCvt_j(g_hi) (g vanishes from 2^p + 2^j up: the product's length)
template <typename T>
static gf2x_status run_icvt_split(const CvtSplit& S, T* data, int smc, cudaStream_t st) {
    gf2x_status s;
    if ((s = run_cvt<T>(S.lo, data, S.p, 1, true, smc, st)) != GF2X_OK) return s;
    if ((s = run_cvt<T>(S.hi, data + (1ull << S.p), S.j, 1, true, smc, st)) != GF2X_OK) return s;
    return launch_shift_xor<T>(data, S.p, 1ull << S.j, smc, st);
}

// tensor map over an FFT pass's output for its TMA tile stores (k_fft2, p.st_tma): tower elements as two 64-bit
// elements; dims (the 2^c-unit column run, middle bits [c, k_lo), rows [k_lo, k_hi), the rest incl. pairs)
static bool make_fft_tmap(const FftParams& q, uint64_t N, CUtensorMap* tm, const void* base = nullptr) {
    auto fn = tmap_encode_fn();
    if (!fn) return false;
    const int R = q.k_hi - q.k_lo;
    const uint64_t total = N * q.batch;
    if (!base) base = q.dst;
    if (q.c > 7 || R > 8 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t dims[4] = {(cuuint64_t)2 << q.c, (cuuint64_t)1 << (q.k_lo - q.c), (cuuint64_t)1 << R, (cuuint64_t)(total >> q.k_hi)};
    cuuint64_t strides[3] = {((cuuint64_t)1 << q.c) * 16, ((cuuint64_t)1 << q.k_lo) * 16, ((cuuint64_t)1 << q.k_hi) * 16};
    cuuint32_t box[4] = {(cuuint32_t)2 << q.c, 1, (cuuint32_t)1 << R, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static gf2x_status launch_fft(const FftPass& f, bool inv, bool psi, const void* src, uint64_t src_per, uint4* dst,
                              const Plan& P, DeviceState* ds, cudaStream_t st, int operands = 1, IdxMap map = {0, 0, 0},
                              uint4* red_dst = nullptr, const uint32_t* red_c = nullptr) {
    FftParams prm;
    prm.red_dst = nullptr;
    if (red_dst) {   // fused Reduce (trunc.cuh): the kernel's fold assumes this geometry
        if (!(psi || inv) || f.c != 5 || f.k_hi - f.k_lo != 6 || FFT_THREADS != 256 || P.batch * operands != 1)
            return fail(GF2X_EINVAL, "fused Reduce geometry");
        prm.red_dst = red_dst;
        for (int i = 0; i < 6; i++) prm.red_c[i] = red_c[i];
    }
    prm.map = map;
    prm.src = src; prm.dst = dst; prm.tabs = ds->tabs;
    prm.src_per = src_per; prm.batch = P.batch * operands;
    prm.m = P.m; prm.c = f.c; prm.k_lo = f.k_lo; prm.k_hi = f.k_hi;
    const int R = f.k_hi - f.k_lo;
    const uint64_t ntiles = (P.N >> (f.c + R)) * prm.batch;
    prm.db = fft2_db(f.c, R, psi) ? 1 : 0;
    prm.wt_shared = fft2_wt_shared(f.c, R, psi) ? 1 : 0;
    const size_t sm = fft2_smem(f.c, R, psi, prm.wt_shared != 0, prm.db != 0, red_dst != nullptr);
    const int occ = sm > 113 * 1024 ? 1 : 2;   // registers (128 x 256 threads) allow at most 2 CTAs/SM
    const int grid = grid_for(ntiles, 1, ds->sm_count, occ);
    const double bytes = (double)prm.batch * (psi ? (double)src_per * 8 : (double)P.N * 16) + (double)prm.batch * P.N * 16;
    const double bfly = (double)prm.batch * (double)(P.N / 2) * R;
    ProfScope ps(inv ? "k_fft<inv>" : (psi ? "k_fft<psi>" : "k_fft"), bytes, st, bfly * OPS_M4R_BUTTERFLY);
    // passes holding the top layer skip the multiplier-0 blocks (a third of their butterflies at 6 layers);
    // elsewhere the check costs more than it saves
    const bool zs = f.k_hi == P.m && !map.bits;
    CUtensorMap tm;
    // TMA tile stores (k_fft2): 1 = double-buffered non-PSI passes (measured c4b 0.571 -> 0.534 ms forward,
    // 0.284 -> 0.267 ms inverse per pass), 2 = also the changeRepr pass (0.604 -> 0.583 ms)
    static const int fft_st = env_int("GF2X_FFT_ST", 2, 0, 2);
    prm.st_tma = (((fft_st >= 1 && !psi && prm.db) || (fft_st >= 2 && psi)) && make_fft_tmap(prm, P.N, &tm)) ? 1 : 0;
    if (!prm.st_tma) memset(&tm, 0, sizeof(tm));
    CUtensorMap tm_src;
    // TMA tile loads (with the stores; non-PSI passes): c4b forward 0.532 -> 0.514 ms, inverse 0.258 -> 0.248 ms
    static const int fft_ld = env_int("GF2X_FFT_LD", 1, 0, 1);
    prm.ld_tma = (fft_ld && prm.st_tma && !psi && prm.db && make_fft_tmap(prm, P.N, &tm_src, src)) ? 1 : 0;
    if (!prm.ld_tma) memset(&tm_src, 0, sizeof(tm_src));
    if (inv) { if (zs) k_fft2<true, false, true><<<grid, FFT_THREADS, sm, st>>>(prm, tm, tm_src); else k_fft2<true, false, false><<<grid, FFT_THREADS, sm, st>>>(prm, tm, tm_src); }
    else if (psi) { if (zs) k_fft2<false, true, true><<<grid, FFT_THREADS, sm, st>>>(prm, tm, tm_src); else k_fft2<false, true, false><<<grid, FFT_THREADS, sm, st>>>(prm, tm, tm_src); }
    else { if (zs) k_fft2<false, false, true><<<grid, FFT_THREADS, sm, st>>>(prm, tm, tm_src); else k_fft2<false, false, false><<<grid, FFT_THREADS, sm, st>>>(prm, tm, tm_src); }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("fft launch: ") + cudaGetErrorString(e));
    return GF2X_OK;
}

// BasisCvt of operand a (or b), split per R22 when planned
static gf2x_status run_cvt_operand(const Plan& P, bool is_a, uint64_t* S, int smc, cudaStream_t st) {
    const CvtSplit& sp = is_a ? P.sa : P.sb;
    if (sp.p >= 0) return run_cvt_fwd_split(sp, S, is_a ? P.na : P.nb, smc, st);
    return run_cvt<uint64_t>(is_a ? P.cvt_a : P.cvt_b, S, is_a ? P.ma : P.mb, P.batch, false, smc, st);
}

// stop_stage: 0 = full product; 1..5 = stop after that stage (debug), result left in Wa
static gf2x_status run_pipeline(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                const Plan& P, void* ws, DeviceState* ds, cudaStream_t st, int stop_stage) {
    unsigned char* base = reinterpret_cast<unsigned char*>(ws);
    uint64_t* Sa = reinterpret_cast<uint64_t*>(base + P.off_sa);
    uint64_t* Sb = reinterpret_cast<uint64_t*>(base + P.off_sb);
    uint4* Wa = reinterpret_cast<uint4*>(base + P.off_wa);
    uint4* Wb = reinterpret_cast<uint4*>(base + P.off_wb);
    const int smc = ds->sm_count;
    gf2x_status s;
    // Split (fused into the first conversion pass when that pass reads the operands itself)
    const bool fused = split_fused(P);
    if (!fused) {
        {
            ProfScope ps("k_prep", (double)P.batch * (P.na + (1ull << P.ma)) * 8, st);
            k_prep<<<grid_for((1ull << P.ma) * P.batch, 256, smc, 8), 256, 0, st>>>(a, P.na, a_bits, P.ma, P.batch, Sa);
        }
        {
            ProfScope ps("k_prep", (double)P.batch * (P.nb + (1ull << P.mb)) * 8, st);
            k_prep<<<grid_for((1ull << P.mb) * P.batch, 256, smc, 8), 256, 0, st>>>(b, P.nb, b_bits, P.mb, P.batch, Sb);
        }
    }
    // BasisCvt on 64-bit blocks
    // Sb | Wb directly follow Sa | Wa: one launch per pass for both operands
    const bool same = (P.ma == P.mb) && P.off_sb == P.off_sa + (1ull << P.ma) * P.batch * 8;
    if (fused) {
        const CvtSrc src{a, b, P.batch, P.na, a_bits};
        if ((s = run_cvt<uint64_t>(P.cvt_a, Sa, P.ma, 2 * P.batch, false, smc, st, &src)) != GF2X_OK) return s;
    } else if (same && P.sa.p < 0 && P.sb.p < 0) {
        if ((s = run_cvt<uint64_t>(P.cvt_a, Sa, P.ma, 2 * P.batch, false, smc, st)) != GF2X_OK) return s;
    } else {
        if ((s = run_cvt_operand(P, true, Sa, smc, st)) != GF2X_OK) return s;
        if ((s = run_cvt_operand(P, false, Sb, smc, st)) != GF2X_OK) return s;
    }
    // changeRepr + FFT_LCH top layers (direct passes; the last planned pass is the bottom one)
    const size_t ndirect = P.fft.size() - 1;
    for (size_t i = 0; i < ndirect; i++) {
        const bool first = (i == 0);
        FftPass f = P.fft[i];
        if (stop_stage == 1) {  // changeRepr only
            if (!first) break;
            f.k_lo = f.k_hi;
        }
        if (same) {   // Wa|Wb and Sa|Sb are contiguous: 2*batch products in one launch
            if ((s = launch_fft(f, false, first, first ? (const void*)Sa : Wa, first ? (1ull << P.ma) : P.N, Wa, P, ds, st, 2)) != GF2X_OK) return s;
        } else {
            if ((s = launch_fft(f, false, first, first ? (const void*)Sa : Wa, first ? (1ull << P.ma) : P.N, Wa, P, ds, st)) != GF2X_OK) return s;
            if ((s = launch_fft(f, false, first, first ? (const void*)Sb : Wb, first ? (1ull << P.mb) : P.N, Wb, P, ds, st)) != GF2X_OK) return s;
        }
    }
    if (ndirect == 0) {  // m <= bot: changeRepr alone (a direct pass with no layers)
        FftPass f{P.m < 5 ? P.m : 5, P.m, P.m, false, 0};
        if (same) {
            if ((s = launch_fft(f, false, true, Sa, 1ull << P.ma, Wa, P, ds, st, 2)) != GF2X_OK) return s;
        } else {
            if ((s = launch_fft(f, false, true, Sa, 1ull << P.ma, Wa, P, ds, st)) != GF2X_OK) return s;
            if ((s = launch_fft(f, false, true, Sb, 1ull << P.mb, Wb, P, ds, st)) != GF2X_OK) return s;
        }
    }
    if (stop_stage == 1) return GF2X_OK;
    // bottom FFT layers of a and b + pointmul + bottom iFFT layers, fused and bit-sliced
    {
        BottomParams bp;
        bp.A = Wa; bp.B = Wb;
        bp.total = P.N * P.batch;
        bp.ntiles = (bp.total + (1ull << BT_BITS) - 1) >> BT_BITS;
        bp.m = P.m; bp.L = P.fft.back().layers;
        bp.map = IdxMap{0, 0, 0};
        bp.mode = stop_stage == 2 ? 1 : (stop_stage == 3 ? 3 : 7);
        ProfScope ps("k_bottom", 48.0 * P.N * P.batch, st, bottom_alu_ops(bp));
        bottom_launch(bp, smc, st);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("bottom launch: ") + cudaGetErrorString(e));
    }
    if (stop_stage == 2 || stop_stage == 3) return GF2X_OK;
    // iFFT_LCH top layers (direct passes in reverse order)
    for (size_t i = ndirect; i-- > 0;) {
        if ((s = launch_fft(P.fft[i], true, false, Wa, P.N, Wa, P, ds, st)) != GF2X_OK) return s;
    }
    if (stop_stage == 4) return GF2X_OK;
    if (stop_stage == 0 && mcomb_ok(P) && ((uintptr_t)c & 15) == 0) {   // (16-byte aligned: TMA / bulk copies in place)
        // R28: changeRepr^-1 and the combine written in the novel basis (64-bit words, into the output), then
        // iBasisCvt of those words in place: the product
        {
            const uint64_t n_write = P.N * P.batch;
            ProfScope ps("k_ipsi_mcomb", 16.0 * n_write + 8.0 * n_write, st);
            k_ipsi_bs<true><<<grid_for(n_write / IB_TILE, 1, smc, 2), IB_THREADS, 6 * IB_TILE * 4, st>>>(
                Wa, ds->tabs, P.N, P.batch, c, nullptr, n_write, ~0ull, ipsi_l2pf());
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("mcomb launch: ") + cudaGetErrorString(e));
        }
        return run_cvt<uint64_t>(P.icvt64, c, P.m, P.batch, true, smc, st);
    }
    // iBasisCvt (tower); the novel coefficients beyond the product's length are zero (R22 split)
    if (P.ic.p >= 0) s = run_icvt_split(P.ic, Wa, smc, st);
    else s = run_cvt<uint4>(P.icvt, Wa, P.m, P.batch, true, smc, st);
    if (s != GF2X_OK) return s;
    if (stop_stage == 5) return GF2X_OK;
    // changeRepr^-1 + InterleavedCombine
    {
        const uint64_t n_out = P.na + P.nb;
        const uint64_t total = n_out * P.batch;
        // bit-sliced when the output is whole tiles of the flat spectrum: n_out = N (any batch), or one
        // product with n_out <= N (the trailing words of the last tile are not written)
        const bool bs = (P.N * P.batch) % IB_TILE == 0 && (n_out == P.N || (P.batch == 1 && n_out < P.N));
        if (bs && !env_flag("GF2X_NO_IPSI_BS")) {
            const uint64_t n_write = n_out == P.N ? P.N * P.batch : n_out;
            ProfScope ps("k_ipsi_bs", 16.0 * n_write + 8.0 * total, st);
            k_ipsi_bs<false><<<grid_for((n_write + IB_TILE - 1) / IB_TILE, 1, smc, 2), IB_THREADS, 6 * IB_TILE * 4, st>>>(
                Wa, ds->tabs, P.N, P.batch, c, nullptr, n_write);
        } else {
            ProfScope ps("k_ipsi_combine", 16.0 * P.N * P.batch + 8.0 * total, st);
            k_ipsi_combine<<<grid_for(total, 256, smc, 2), 256, 16 * 256 * 16, st>>>(Wa, ds->tabs, P.N, n_out, P.batch, c, nullptr);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("combine launch: ") + cudaGetErrorString(e));
    }
    return GF2X_OK;
}

static bool overlaps(const void* p, size_t pb, const void* q, size_t qb) {
    const char* a = (const char*)p;
    const char* b = (const char*)q;
    return a < b + qb && b < a + pb;
}

// Per-(device, stream) workspace cache shared by every entry point.  It only grows; a buffer it
// outgrows is retired, not freed, because a CUDA graph captured earlier may still reference it
// (retired buffers are freed by gf2x_release).  Growing during stream capture is an error: the
// allocation would not be part of the graph and a later growth would leave the graph pointing at
// a retired buffer of the wrong size -- warm up at the largest size first, or pass a workspace
// (gf2x_mul_ws).
static gf2x_status stream_workspace(DeviceState* ds, cudaStream_t st, size_t bytes, void** out) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& ent = ds->ws[st];
    if (ent.second < bytes) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return fail(GF2X_ECUDA, "cudaStreamIsCapturing failed");
        if (cs != cudaStreamCaptureStatusNone)
            return fail(GF2X_EINVAL, "the stream's workspace must grow while the stream is being captured: run the "
                                     "call once before capture (or use gf2x_mul_ws with a caller-owned workspace)");
        if (ent.first) ds->retired.push_back(ent.first);
        ent.first = nullptr;
        ent.second = 0;
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) return fail(GF2X_ENOMEM, std::string("workspace: ") + cudaGetErrorString(e));
        ent.first = p;
        ent.second = bytes;
    }
    *out = ent.first;
    return GF2X_OK;
}

// ------------------------------------------------------------------------------ the fused small-N kernel
// 0: not used; else the cluster size of k_small (small.cuh): products of N = 2^m points, 5 <= m <= 11
static int small_cluster(const Plan& P) {
    if (P.m < 5 || P.m > 11 || env_flag("GF2X_NO_SMALL")) return 0;
    std::vector<CvtOp> oa, ob, oi;
    cvt_ops(P.ma, 0, oa);
    cvt_ops(P.mb, 0, ob);
    cvt_ops(P.m, 0, oi);
    if (oa.size() > SM_MAX_OPS || ob.size() > SM_MAX_OPS || oi.size() > SM_MAX_OPS) return 0;
    if (P.batch == 1 && P.m >= 7) {   // one product: its limbs on four CTAs, with m >= 9 (8) also its points on
        // four (two) segments: 16 (8) CTAs; GF2X_SMALL_CL = 4 / 8 / 16 caps the cluster
        const int cap = env_int("GF2X_SMALL_CL", 16, 4, 16);
        if (cap >= 16 && P.m >= 9) return 16;
        if (cap >= 8 && P.m >= 8) return 8;
        return 4;
    }
    // batches keep the multi-pass path: one CTA per 2^9-point product measured 1.12 ms at c2 against 0.56
    // (per-butterfly constants and M4R-4 changeRepr^-1 lookups cost more than the bit-sliced bottom kernel);
    // GF2X_SMALL_BATCH=1 selects it (tested)
    if (P.batch > 1 && env_flag_now("GF2X_SMALL_BATCH")) return small_layout(P.m, 1).total * 4 <= 200 * 1024 ? 1 : (P.m >= 7 ? 4 : 0);
    return 0;
}

// The FFT constants of k_small (small.cuh KT) for 2^m points cut into 2^QB segments, every segment's table
// (ktw words each, 16-byte multiples): K_b = c v_b for each local layer and block, c = s_k(block base) the XOR
// of S[k][j] over the base's bits (layer_const), computed on the host once per device and (m, QB) like the
// App. C constants (frob.cuh); the kernel copies its segment's table with cp.async instead of building it.
// (*out = nullptr when the table is not built yet and `build` is false: the kernel then builds its own)
static gf2x_status get_small_kt(DeviceState* ds, int m, int QB, bool build, const uint32_t** out, uint32_t* ktw) {
    const int mloc = m - QB;
    *ktw = (kt_off(m, mloc, mloc) + 3) & ~3u;
    std::lock_guard<std::mutex> lk(g_mu);
    const int key = m * 4 + QB;
    auto it = ds->small_kt.find(key);
    if (it != ds->small_kt.end()) { *out = it->second; return GF2X_OK; }
    *out = nullptr;
    if (!build) return GF2X_OK;
    const uint32_t seg = 1u << mloc, QC = 1u << QB;
    std::vector<uint32_t> h((size_t)QC * *ktw, 0u);
    for (uint32_t q = 0; q < QC; q++)
        for (int k = 0; k < mloc; k++) {
            const int W = sm_width(m - k);
            for (uint32_t blk = 0; blk < (seg >> (k + 1)); blk++) {
                uint32_t bb = (q * seg + (blk << (k + 1))) >> (k + 1), cst = 0;
                for (int j = k + 1; bb; bb >>= 1, j++)
                    if (bb & 1) cst ^= ds->host->S[k * 32 + j];
                uint32_t K[16];
                if (W == 2) sm_consts<2>(cst, K);
                else if (W == 4) sm_consts<4>(cst, K);
                else if (W == 8) sm_consts<8>(cst, K);
                else sm_consts<16>(cst, K);
                uint32_t* d = h.data() + (size_t)q * *ktw + kt_off(m, mloc, k) + blk * W;
                for (int b = 0; b < W; b++) d[b] = K[b];
            }
        }
    uint32_t* d = nullptr;
    if (cudaMalloc(&d, h.size() * 4) != cudaSuccess) return fail(GF2X_ENOMEM, "k_small constants");
    if (cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return fail(GF2X_ECUDA, "k_small constants");
    }
    ds->small_kt[key] = d;
    *out = d;
    return GF2X_OK;
}

static gf2x_status run_small(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                             const Plan& P, int CL, DeviceState* ds, cudaStream_t st) {
    if (CL == 16) {   // a 16-CTA cluster is non-portable: fall back to 8 where the device cannot hold one
        static int ok16[64];   // per device: 0 unknown, 1 yes, 2 no
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64 && ok16[dev] == 0) {
            cudaLaunchConfig_t q;
            memset(&q, 0, sizeof(q));
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 16;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            q.attrs = at;
            q.numAttrs = 1;
            q.blockDim = dim3(SM_THREADS);
            q.gridDim = dim3(16);
            q.dynamicSmemBytes = (size_t)small_layout(P.m, 16, true).total * 4;
            int ncl = 0;
            const cudaError_t qe = cudaOccupancyMaxActiveClusters(&ncl, k_small<16>, &q);
            if (qe != cudaSuccess) cudaGetLastError();
            ok16[dev] = (qe == cudaSuccess && ncl >= 1) ? 1 : 2;
        }
        if (dev >= 64 || ok16[dev] != 1) CL = 8;
    }
    SmallParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.a = a; sp.b = b; sp.c = c;
    sp.na = P.na; sp.nb = P.nb; sp.a_bits = a_bits; sp.b_bits = b_bits; sp.batch = P.batch;
    sp.m = P.m; sp.ma = P.ma; sp.mb = P.mb;
    std::vector<CvtOp> oa, ob, oi;
    cvt_ops(P.ma, 0, oa);
    cvt_ops(P.mb, 0, ob);
    cvt_ops(P.m, 0, oi);
    sp.nops_a = (int)oa.size(); sp.nops_b = (int)ob.size(); sp.nops_i = (int)oi.size();
    for (size_t i = 0; i < oa.size(); i++) sp.ops_a[i] = oa[i];
    for (size_t i = 0; i < ob.size(); i++) sp.ops_b[i] = ob[i];
    for (size_t i = 0; i < oi.size(); i++) sp.ops_i[i] = oi[i];
    sp.tabs = ds->tabs;
    // split conversions (small.cuh sm_conv_op / sm_low_block): op list idx of 2^mm units -> top-run and
    // low-block lengths and the low block's window bits K (split only when the windows fit a point segment)
    auto seg_cvt = [&](int mm, int idx) {
        sp.split[idx] = 0; sp.ntop[idx] = 0; sp.nlow[idx] = 0; sp.kw[idx] = 0;
        if (mm <= 2 || env_flag_now("GF2X_SMALL_NO_SEGCVT")) return;
        int K = 1;
        while (2 * K <= mm - 1) K *= 2;   // (cvt_ops' split)
        if (K > P.m - small_qb(CL)) return;
        std::vector<CvtOp> low;
        cvt_ops(K, 0, low);
        sp.split[idx] = 1; sp.ntop[idx] = mm - K; sp.nlow[idx] = (int)low.size(); sp.kw[idx] = K;
    };
    seg_cvt(P.ma, 0);
    seg_cvt(P.mb, 1);
    seg_cvt(P.m, 2);
    // the segment's FFT constants precomputed per CTA when they fit (GF2X_SMALL_NO_KT=1: per layer and thread)
    sp.kt = !env_flag_now("GF2X_SMALL_NO_KT") && (size_t)small_layout(P.m, CL, true).total * 4 <= 220 * 1024;
    sp.ktg = nullptr;
    sp.ktw = 0;
    if (sp.kt && !env_flag_now("GF2X_SMALL_KT_BUILD")) {   // (GF2X_SMALL_KT_BUILD=1: every CTA builds its table)
        // (no allocation or copy while the stream is being captured into a graph: the kernel builds its table)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        gf2x_status ks = get_small_kt(ds, P.m, small_qb(CL), cs == cudaStreamCaptureStatusNone, &sp.ktg, &sp.ktw);
        if (ks != GF2X_OK) return ks;
    }
    const size_t sm = (size_t)small_layout(P.m, CL, sp.kt != 0).total * 4;
    const double bytes = (double)P.batch * 8.0 * (P.na + P.nb + P.na + P.nb);
    ProfScope ps(CL == 1 ? "k_small<1>" : (CL == 4 ? "k_small<4>" : (CL == 8 ? "k_small<8>" : "k_small<16>")), bytes, st);
    cudaError_t e;
    if (CL == 1) {
        const int occ = std::max(1, (int)(220 * 1024 / (sm + 1024)));
        k_small<1><<<grid_for(P.batch, 1, ds->sm_count, occ), SM_THREADS, sm, st>>>(sp);
        e = cudaGetLastError();
    } else {
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof(cfg));
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.blockDim = dim3(SM_THREADS);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        const uint64_t ncl = std::min<uint64_t>(P.batch, (uint64_t)(ds->sm_count / CL) * std::max(1, (int)(220 * 1024 / (sm + 1024))));
        cfg.gridDim = dim3((unsigned)(CL * ncl));
        e = cudaLaunchKernelEx(&cfg, CL == 4 ? k_small<4> : (CL == 8 ? k_small<8> : k_small<16>), sp);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    return e == cudaSuccess ? GF2X_OK : fail(GF2X_ECUDA, std::string("small launch: ") + cudaGetErrorString(e));
}

static gf2x_status run_pipeline_a4(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                   const Plan& P, void* ws, DeviceState* ds, cudaStream_t st, int stop_stage);
static int run_trunc_if_eligible(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                 const Plan& P, void* ws, DeviceState* ds, cudaStream_t st, gf2x_status* out);
// algo: 5 = Alg. 5 (the product path), 4 = Alg. 4 (comparison variant, alg4.cuh)
static gf2x_status mul_common(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                              int64_t batch, void* user_ws, size_t user_ws_bytes, void* stream, int stop_stage,
                              uint64_t* stage_out, int algo = 5) {
    if (batch < 0) return fail(GF2X_EINVAL, "negative batch");
    if (batch == 0) return GF2X_OK;
    const uint64_t na = (a_bits + 63) / 64, nb = (b_bits + 63) / 64;
    const size_t out_bytes = (size_t)(na + nb) * 8 * (size_t)batch;
    if (!c && out_bytes && !stop_stage) return fail(GF2X_EINVAL, "null output");
    if ((!a && na) || (!b && nb)) return fail(GF2X_EINVAL, "null input");
    if (c && out_bytes && ((a && overlaps(c, out_bytes, a, na * 8 * batch)) || (b && overlaps(c, out_bytes, b, nb * 8 * batch))))
        return fail(GF2X_EINVAL, "output overlaps an input");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (a_bits == 0 || b_bits == 0) {
        if (out_bytes) CUDA_TRY(cudaMemsetAsync(c, 0, out_bytes, st));
        return GF2X_OK;
    }
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    Plan P;
    if ((s = make_plan(a_bits, b_bits, batch, P)) != GF2X_OK) return s;
    // products of at most 2^11 points: the fused single-kernel pipeline (no workspace)
    if (algo == 5 && !stop_stage) {
        const int CL = small_cluster(P);
        if (CL) return run_small(a, a_bits, b, b_bits, c, P, CL, ds, st);
    }
    void* ws = user_ws;
    if (ws) {
        if (user_ws_bytes < P.bytes) return fail(GF2X_ENOMEM, "workspace too small");
    } else {
        if ((s = stream_workspace(ds, st, P.bytes, &ws)) != GF2X_OK) return s;
    }
    // products just above a power of two take the truncated FFT (trunc.cuh) unless a stage is requested
    if (algo == 5 && !stop_stage && run_trunc_if_eligible(a, a_bits, b, b_bits, c, P, ws, ds, st, &s)) return s;
    s = algo == 4 ? run_pipeline_a4(a, a_bits, b, b_bits, c, P, ws, ds, st, stop_stage)
                  : run_pipeline(a, a_bits, b, b_bits, c, P, ws, ds, st, stop_stage);
    if (s != GF2X_OK) return s;
    if (stop_stage && stage_out) {
        CUDA_TRY(cudaMemcpyAsync(stage_out, reinterpret_cast<unsigned char*>(ws) + P.off_wa, P.N * 16,
                                 cudaMemcpyDeviceToDevice, st));
    }
    return GF2X_OK;
}

#include "shard.cuh"
#include "w128.cuh"
#include "alg4.cuh"
#include "trunc.cuh"
#include "frob.cuh"

extern "C" {

gf2x_status gf2x_mul(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c, void* stream) {
    return mul_common(a, a_bits, b, b_bits, c, 1, nullptr, 0, stream, 0, nullptr);
}

gf2x_status gf2x_mul_batched(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                             int64_t batch, void* stream) {
    return mul_common(a, a_bits, b, b_bits, c, batch, nullptr, 0, stream, 0, nullptr);
}

size_t gf2x_workspace_bytes(uint64_t a_bits, uint64_t b_bits, int64_t batch) {
    if (a_bits == 0 || b_bits == 0 || batch <= 0) return 0;
    Plan P;
    if (make_plan(a_bits, b_bits, batch, P) != GF2X_OK) return 0;
    return P.bytes;
}

gf2x_status gf2x_mul_ws(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                        int64_t batch, void* ws, size_t ws_bytes, void* stream) {
    if (!ws) return fail(GF2X_EINVAL, "null workspace");
    return mul_common(a, a_bits, b, b_bits, c, batch, ws, ws_bytes, stream, 0, nullptr);
}

int gf2x_launch_count(uint64_t a_bits, uint64_t b_bits, int64_t batch) {
    if (a_bits == 0 || b_bits == 0 || batch <= 0) return 0;
    Plan P;
    if (make_plan(a_bits, b_bits, batch, P) != GF2X_OK) return 0;
    TruncGeom TG;
    if (trunc_geom(P, TG)) return launches_of_trunc(P, TG);
    return launches_of(P);
}

gf2x_status gf2x_debug_stage(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, int stage,
                             uint64_t* out, void* stream) {
    if (stage < 1 || stage > 5 || !out || a_bits == 0 || b_bits == 0) return fail(GF2X_EINVAL, "bad debug stage request");
    return mul_common(a, a_bits, b, b_bits, nullptr, 1, nullptr, 0, stream, stage, out);
}

gf2x_status gf2x_mul_w(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c, int64_t batch,
                       int w, void* stream) {
    if (w == 64) return mul_common(a, a_bits, b, b_bits, c, batch, nullptr, 0, stream, 0, nullptr);
    if (w == 128) return mul_common_w128(a, a_bits, b, b_bits, c, batch, stream, 0, nullptr);
    return fail(GF2X_EINVAL, "block width w must be 64 or 128");
}

int gf2x_launch_count_w(uint64_t a_bits, uint64_t b_bits, int64_t batch, int w) {
    if (w == 64) return gf2x_launch_count(a_bits, b_bits, batch);
    if (w != 128 || batch <= 0) return 0;
    if (a_bits == 0 || b_bits == 0) return 1;
    PlanW128 P;
    if (make_plan_w128(a_bits, b_bits, batch, P) != GF2X_OK) return -1;
    return launches_of_w128(P);
}

gf2x_status gf2x_debug_stage_w128(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, int stage,
                                  uint64_t* out, void* stream) {
    if (stage != 1 && stage != 2 && stage != 3 && stage != 5) return fail(GF2X_EINVAL, "stage must be 1, 2, 3 or 5");
    if (!out || a_bits == 0 || b_bits == 0) return fail(GF2X_EINVAL, "null output or empty operand");
    return mul_common_w128(a, a_bits, b, b_bits, nullptr, 1, stream, stage, out);
}

gf2x_status gf2x_mul_alg4(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                          int64_t batch, void* stream) {
    return mul_common(a, a_bits, b, b_bits, c, batch, nullptr, 0, stream, 0, nullptr, 4);
}

gf2x_status gf2x_debug_stage_alg4(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, int stage,
                                  uint64_t* out, void* stream) {
    if (stage != 2 && stage != 3) return fail(GF2X_EINVAL, "stage must be 2 or 3");
    if (!out || a_bits == 0 || b_bits == 0) return fail(GF2X_EINVAL, "null output or empty operand");
    return mul_common(a, a_bits, b, b_bits, nullptr, 1, nullptr, 0, stream, stage, out, 4);
}

gf2x_status gf2x_mul_frob(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c, void* stream) {
    if ((a_bits && !a) || (b_bits && !b) || !c) return fail(GF2X_EINVAL, "null pointer");
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    return run_frob_mul(a, a_bits, b, b_bits, c, ds, (cudaStream_t)stream);
}

gf2x_status gf2x_basis_cvt_bits(uint64_t* words, int M, int inverse, void* stream) {
    if (!words || M < 6 || M > 40) return fail(GF2X_EINVAL, "bit-level BasisCvt needs 6 <= M <= 40 and a buffer");
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    return run_bitcvt(words, M, inverse != 0, ds->sm_count, (cudaStream_t)stream);
}

gf2x_status gf2x_comm_unique_id(void* id_out) {
    if (!id_out) return fail(GF2X_EINVAL, "null id buffer");
    std::string err = nccl_load();
    if (!err.empty()) return fail(GF2X_ENCCL, err);
    nccl_uid_t id;
    int rc = g_nccl.GetUniqueId(&id);
    if (rc) return fail(GF2X_ENCCL, std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(rc));
    memcpy(id_out, &id, sizeof(id));
    return GF2X_OK;
}

gf2x_status gf2x_comm_init(const void* nccl_unique_id, int nranks, int rank, gf2x_comm_t* out) {
    if (!nccl_unique_id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(GF2X_EINVAL, "bad comm arguments");
    std::string err = nccl_load();
    if (!err.empty()) return fail(GF2X_ENCCL, err);
    nccl_uid_t id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    if (nranks > SHARD_MAXG) return fail(GF2X_EINVAL, "at most 8 ranks");
    gf2x_comm_s* c = new gf2x_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    c->ws = nullptr;
    c->ws_bytes = 0;
    c->p2p = 0;
    c->aborted = 0;
    for (int r = 0; r < SHARD_MAXG; r++) c->peer_ws[r] = nullptr;
    cudaGetDevice(&c->device);
    if (cudaMalloc(&c->d_sync, 256 + SHARD_MAXG * sizeof(cudaIpcMemHandle_t)) != cudaSuccess) {
        delete c;
        return fail(GF2X_ENOMEM, "comm sync buffer");
    }
    cudaMemset(c->d_sync, 0, 256);
    int rc = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
    if (rc) {
        delete c;
        return fail(GF2X_ENCCL, std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(rc));
    }
    *out = c;
    return GF2X_OK;
}

gf2x_status gf2x_comm_init_host(int nranks, int rank, gf2x_host_barrier_fn barrier, gf2x_host_allgather_fn allgather,
                                void* user, gf2x_comm_t* out) {
    if (!out || !barrier || !allgather || nranks < 1 || rank < 0 || rank >= nranks) return fail(GF2X_EINVAL, "bad comm arguments");
    if (nranks > SHARD_MAXG) return fail(GF2X_EINVAL, "at most 8 ranks");
    gf2x_comm_s* c = new gf2x_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    c->comm = nullptr;
    c->ws = nullptr;
    c->ws_bytes = 0;
    c->p2p = 0;
    c->aborted = 0;
    c->host = 1;
    c->hbar = barrier;
    c->hag = allgather;
    c->huser = user;
    for (int r = 0; r < SHARD_MAXG; r++) c->peer_ws[r] = nullptr;
    cudaGetDevice(&c->device);
    if (cudaMalloc(&c->d_sync, 256 + SHARD_MAXG * sizeof(cudaIpcMemHandle_t)) != cudaSuccess) {
        delete c;
        return fail(GF2X_ENOMEM, "comm sync buffer");
    }
    *out = c;
    return GF2X_OK;
}

static void comm_unmap_peers(gf2x_comm_s* c) {
    for (int r = 0; r < SHARD_MAXG; r++)
        if (c->peer_ws[r] && r != c->rank) cudaIpcCloseMemHandle(c->peer_ws[r]);
    for (int r = 0; r < SHARD_MAXG; r++) c->peer_ws[r] = nullptr;
    c->p2p = 0;
}

// Map every rank's workspace into this process (CUDA IPC; NVLink peer access).  Collective: the handles
// go around with an NCCL all-gather and the outcome is agreed with an all-reduce(min), so every rank
// takes the same exchange path.  GF2X_SHARD_NCCL=1 keeps NCCL send/recv.
static gf2x_status comm_map_peers_host(gf2x_comm_s* c, cudaStream_t st) {
    comm_unmap_peers(c);
    const int G = c->nranks;
    CUDA_TRY(cudaStreamSynchronize(st));
    cudaIpcMemHandle_t mine;
    memset(&mine, 0, sizeof(mine));
    int ok = cudaIpcGetMemHandle(&mine, c->ws) == cudaSuccess ? 1 : 0;
    if (!ok) cudaGetLastError();
    std::vector<cudaIpcMemHandle_t> hs(G);
    if (c->hag(&mine, hs.data(), sizeof(mine), c->huser) != 0) return fail(GF2X_ENCCL, "host all-gather callback failed");
    c->peer_ws[c->rank] = c->ws;
    for (int r = 0; r < G && ok; r++) {
        if (r == c->rank) continue;
        if (cudaIpcOpenMemHandle(&c->peer_ws[r], hs[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            ok = 0;
            c->peer_ws[r] = nullptr;
            cudaGetLastError();
        }
    }
    std::vector<int> oks(G);
    if (c->hag(&ok, oks.data(), sizeof(int), c->huser) != 0) return fail(GF2X_ENCCL, "host all-gather callback failed");
    for (int r = 0; r < G; r++) ok = std::min(ok, oks[r]);
    if (!ok) {
        comm_unmap_peers(c);
        return fail(GF2X_ECUDA, "host-mode communicator: CUDA IPC mapping of the peers' workspaces failed");
    }
    c->p2p = 1;
    return GF2X_OK;
}

static gf2x_status comm_map_peers(gf2x_comm_s* c, cudaStream_t st) {
    if (c->host) return comm_map_peers_host(c, st);
    comm_unmap_peers(c);
    const int G = c->nranks;
    int ok = env_flag_now("GF2X_SHARD_NCCL") ? 0 : 1;
    cudaIpcMemHandle_t mine;
    memset(&mine, 0, sizeof(mine));
    if (ok && cudaIpcGetMemHandle(&mine, c->ws) != cudaSuccess) { ok = 0; cudaGetLastError(); }
    unsigned char* dh = reinterpret_cast<unsigned char*>(c->d_sync) + 256;
    CUDA_TRY(cudaMemcpyAsync(dh + c->rank * sizeof(mine), &mine, sizeof(mine), cudaMemcpyHostToDevice, st));
    int rc = g_nccl.AllGather(dh + c->rank * sizeof(mine), dh, sizeof(mine), NCCL_UINT8, c->comm, st);
    if (rc) return fail(GF2X_ENCCL, std::string("IPC handle all-gather: ") + g_nccl.GetErrorString(rc));
    std::vector<cudaIpcMemHandle_t> hs(G);
    CUDA_TRY(cudaMemcpyAsync(hs.data(), dh, G * sizeof(mine), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    c->peer_ws[c->rank] = c->ws;
    for (int r = 0; r < G && ok; r++) {
        if (r == c->rank) continue;
        if (cudaIpcOpenMemHandle(&c->peer_ws[r], hs[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            ok = 0;
            c->peer_ws[r] = nullptr;
            cudaGetLastError();
        }
    }
    int* dflag = c->d_sync + 1;
    CUDA_TRY(cudaMemcpyAsync(dflag, &ok, sizeof(int), cudaMemcpyHostToDevice, st));
    rc = g_nccl.AllReduce(dflag, dflag, 1, NCCL_INT32, NCCL_MIN, c->comm, st);
    if (rc) return fail(GF2X_ENCCL, std::string("IPC agreement: ") + g_nccl.GetErrorString(rc));
    int all = 0;
    CUDA_TRY(cudaMemcpyAsync(&all, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (!all) comm_unmap_peers(c);
    else c->p2p = 1;
    return GF2X_OK;
}

int gf2x_comm_peer_memory(gf2x_comm_t comm) { return comm ? comm->p2p : -1; }

gf2x_status gf2x_experiment_ipsi_tc(const void* P, uint64_t n, void* out, uint32_t lbo, uint32_t sbo, void* stream) {
    if (!P || !out) return fail(GF2X_EINVAL, "null argument");
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    const uint64_t ntiles = (n + 127) >> 7;
    ProfScope ps("k_ipsi_tc", 32.0 * n, (cudaStream_t)stream);
    k_ipsi_tc<<<grid_for(ntiles, 1, ds->sm_count, env_int("GF2X_TC_OCC", 4, 1, 4)), TC_THREADS, 0, (cudaStream_t)stream>>>(
        (const uint4*)P, n, ds->tabs, (uint4*)out, lbo ? lbo : 128, sbo ? sbo : 1024);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GF2X_OK : fail(GF2X_ECUDA, std::string("ipsi tc launch: ") + cudaGetErrorString(e));
}

gf2x_status gf2x_experiment_fft_low(void* A, void* B, uint32_t m, int variant, void* stream) {
    if (!A || !B || m < 11 || m > 30 || variant < 0 || variant > 1) return fail(GF2X_EINVAL, "fft_low experiment arguments");
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t n = 1ull << m;
    if (variant == 0) {   // k_bottom's bit-sliced layers 4 .. 0 (forward only, both operands)
        BottomParams bp;
        bp.A = (uint4*)A; bp.B = (uint4*)B;
        bp.total = n;
        bp.ntiles = (n + (1ull << BT_BITS) - 1) >> BT_BITS;
        bp.m = (int)m; bp.L = 5;
        bp.map = IdxMap{0, 0, 0};
        bp.mode = 1;
        ProfScope ps("k_bottom<fwd, L=5>", 64.0 * n, st);
        bottom_launch(bp, ds->sm_count, st);
    } else {
        ProfScope ps("k_fft_low_shfl", 64.0 * n, st);
        k_fft_low_shfl<<<ds->sm_count * 4, SHFL_THREADS, 0, st>>>((uint4*)A, (uint4*)B, n);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GF2X_OK : fail(GF2X_ECUDA, std::string("fft_low experiment: ") + cudaGetErrorString(e));
}

gf2x_status gf2x_comm_check(gf2x_comm_t comm) {
    if (!comm) return fail(GF2X_EINVAL, "null communicator");
    return comm_check(comm);
}

gf2x_status gf2x_comm_abort(gf2x_comm_t comm) {
    if (!comm) return fail(GF2X_EINVAL, "null communicator");
    comm_abort(comm, "gf2x_comm_abort");
    return GF2X_OK;
}

gf2x_status gf2x_comm_wait(gf2x_comm_t comm, void* stream, double timeout_s) {
    if (!comm) return fail(GF2X_EINVAL, "null communicator");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        gf2x_status s = comm_check(comm);
        if (s != GF2X_OK) return s;
        const cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) return comm_check(comm);
        if (q != cudaErrorNotReady) return fail(GF2X_ECUDA, std::string("stream: ") + cudaGetErrorString(q));
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (timeout_s > 0 && dt > timeout_s) {
            comm_abort(comm, "gf2x_comm_wait timed out (a peer stopped participating?)");
            return fail(GF2X_ENCCL, comm->abort_reason);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

gf2x_status gf2x_comm_destroy(gf2x_comm_t comm) {
    if (!comm) return GF2X_OK;
    cudaDeviceSynchronize();
    comm_unmap_peers(comm);
    if (comm->d_sync) cudaFree(comm->d_sync);
    if (comm->ws) { cudaDeviceSynchronize(); cudaFree(comm->ws); }
    int rc = (g_nccl.h && comm->comm) ? g_nccl.CommDestroy(comm->comm) : 0;   // (an aborted comm is already gone)
    delete comm;
    if (rc) return fail(GF2X_ENCCL, std::string("ncclCommDestroy: ") + g_nccl.GetErrorString(rc));
    return GF2X_OK;
}

static void rank_bufs(RankCtx& R, unsigned char* base, const ShardGeom& S) {
    for (int b = 0; b < SB_COUNT; b++) R.buf[b] = base + S.off[b];
    R.buf[SB_INA] = (unsigned char*)R.a_shard;
    R.buf[SB_INB] = (unsigned char*)R.b_shard;
}

gf2x_status gf2x_mul_sharded(const uint64_t* a_shard, const uint64_t* b_shard, uint64_t bits, uint64_t* c_shard,
                             gf2x_comm_t comm, void* stream) {
    if (!comm || !a_shard || !b_shard || !c_shard) return fail(GF2X_EINVAL, "null argument");
    gf2x_status s0 = comm_check(comm);   // an earlier asynchronous NCCL failure: do not enqueue on a broken comm
    if (s0 != GF2X_OK) return s0;
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    ShardGeom S;
    if ((s = shard_geom(bits, comm->nranks, S)) != GF2X_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (comm->ws_bytes < S.bytes) {
        // (collective: every rank grows its workspace in the same call, the sizes depend on (bits, G) only)
        cudaDeviceSynchronize();
        comm_unmap_peers(comm);
        if (comm->ws) { cudaFree(comm->ws); comm->ws = nullptr; comm->ws_bytes = 0; }
        cudaError_t e = cudaMalloc(&comm->ws, S.bytes);
        if (e != cudaSuccess) return fail(GF2X_ENOMEM, std::string("shard workspace: ") + cudaGetErrorString(e));
        comm->ws_bytes = S.bytes;
        if ((s = comm_map_peers(comm, st)) != GF2X_OK) return s;
    }
    std::vector<RankCtx> ranks(1);
    ranks[0].r = comm->rank;
    ranks[0].a_shard = a_shard;
    ranks[0].b_shard = b_shard;
    ranks[0].c_shard = c_shard;
    rank_bufs(ranks[0], (unsigned char*)comm->ws, S);
    ShardExec X{false, comm, st, &ranks};
    X.p2p = comm->p2p != 0;
    X.off = S.off;
    for (int r = 0; r < comm->nranks; r++) X.peer[r] = (unsigned char*)comm->peer_ws[r];
    if ((s = run_sharded(S, X, ds, ds->host, bits)) != GF2X_OK) return s;
    // the next call rewrites this workspace: every peer must be done pulling from it
    return X.p2p ? X.barrier() : GF2X_OK;
}

static gf2x_status sharded_sim(const uint64_t* a, const uint64_t* b, uint64_t bits, uint64_t* c, int nranks, void* stream,
                               int debug_stage, uint64_t* dbg) {
    if (!a || !b || (!c && !debug_stage)) return fail(GF2X_EINVAL, "null argument");
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    ShardGeom S;
    if ((s = shard_geom(bits, nranks, S)) != GF2X_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t need = S.bytes * (size_t)nranks;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (ds->shard_ws_bytes < need) {
            if (ds->shard_ws) { cudaDeviceSynchronize(); cudaFree(ds->shard_ws); ds->shard_ws = nullptr; ds->shard_ws_bytes = 0; }
            cudaError_t e = cudaMalloc(&ds->shard_ws, need);
            if (e != cudaSuccess) return fail(GF2X_ENOMEM, std::string("shard sim workspace: ") + cudaGetErrorString(e));
            ds->shard_ws_bytes = need;
        }
    }
    std::vector<RankCtx> ranks(nranks);
    for (int r = 0; r < nranks; r++) {
        ranks[r].r = r;
        ranks[r].a_shard = a + r * (S.n / nranks);
        ranks[r].b_shard = b + r * (S.n / nranks);
        ranks[r].c_shard = c ? c + r * S.Nloc : nullptr;
        rank_bufs(ranks[r], (unsigned char*)ds->shard_ws + r * S.bytes, S);
    }
    ShardExec X{true, nullptr, st, &ranks};
    X.p2p = !env_flag_now("GF2X_SHARD_LISTS");   // default: the peer-memory pulls (lists: copy engine)
    X.off = S.off;
    return run_sharded(S, X, ds, ds->host, bits, debug_stage, (uint4*)dbg);
}

gf2x_status gf2x_mul_sharded_sim(const uint64_t* a, const uint64_t* b, uint64_t bits, uint64_t* c, int nranks, void* stream) {
    return sharded_sim(a, b, bits, c, nranks, stream, 0, nullptr);
}

gf2x_status gf2x_debug_shard_stage(const uint64_t* a, const uint64_t* b, uint64_t bits, int nranks, int stage, uint64_t* out,
                                   void* stream) {
    if ((stage != 1 && stage != 5) || !out) return fail(GF2X_EINVAL, "bad shard debug stage");
    return sharded_sim(a, b, bits, nullptr, nranks, stream, stage, out);
}

int gf2x_plan(uint64_t a_bits, uint64_t b_bits, int64_t batch, char* buf, size_t cap) {
    if (a_bits == 0 || b_bits == 0 || batch < 1) return -1;
    Plan P;
    if (make_plan(a_bits, b_bits, batch, P) != GF2X_OK) return -1;
    auto cvt = [](const std::vector<CvtPass>& v) {
        std::string o = "[";
        for (size_t i = 0; i < v.size(); i++) {
            const CvtPass& p = v[i];
            const char* kind = p.stream ? "stream" : (p.res ? "res" : (p.rb ? "rb" : "tile"));
            o += (i ? ", " : "");
            o += "{\"kind\": \"" + std::string(kind) + "\", \"ops\": [";
            for (size_t j = 0; j < p.ops.size(); j++)
                o += (j ? ", " : "") + std::string("[") + std::to_string(p.ops[j].lg) + ", " + std::to_string(p.ops[j].K) + "]";
            o += "]}";
        }
        return o + "]";
    };
    std::string out = "{\"m\": " + std::to_string(P.m) + ", \"N\": " + std::to_string(P.N) + ", \"ma\": " +
                      std::to_string(P.ma) + ", \"mb\": " + std::to_string(P.mb) + ", \"workspace\": " +
                      std::to_string(P.bytes) + ", \"fft\": [";
    for (size_t i = 0; i + 1 < P.fft.size(); i++)
        out += (i ? ", " : "") + std::string("[") + std::to_string(P.fft[i].c) + ", " + std::to_string(P.fft[i].k_lo) + ", " +
               std::to_string(P.fft[i].k_hi) + "]";
    TruncGeom TG;
    const int tj = trunc_geom(P, TG) ? TG.j : -1;
    out += "], \"bottom\": " + std::to_string(P.fft.back().layers) + ", \"trunc_j\": " + std::to_string(tj) +
           ", \"cvt_a\": " + cvt(P.cvt_a) +
           ", \"cvt_b\": " + cvt(P.cvt_b) + ", \"icvt\": " + cvt(P.icvt);
    auto sp = [](const CvtSplit& S) {
        return S.p < 0 ? std::string("null") : "[" + std::to_string(S.p) + ", " + std::to_string(S.j) + "]";
    };
    out += ", \"split\": {\"a\": " + sp(P.sa) + ", \"b\": " + sp(P.sb) + ", \"icvt\": " + sp(P.ic) + "}}";
    if (buf && cap) {
        const size_t n = std::min(cap - 1, out.size());
        memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return (int)out.size();
}

int gf2x_shard_plan(uint64_t bits, int nranks, char* buf, size_t cap) {
    ShardGeom S;
    if (shard_geom(bits, nranks, S) != GF2X_OK) return -1;
    ShardXfers X;
    shard_xfers(S, X);
    static const char* bn[SB_ALL] = {"A", "B", "W", "T", "X", "HALO", "COPY_A", "COPY_B", "IN_A", "IN_B"};
    auto list = [&](const std::vector<Xfer>& xs) {
        std::string o = "[";
        for (size_t i = 0; i < xs.size(); i++) {
            char t[192];
            snprintf(t, sizeof(t), "%s[%d, %d, \"%s\", \"%s\", %zu, %zu, %zu]", i ? ", " : "", xs[i].src, xs[i].dst,
                     bn[xs[i].sb], bn[xs[i].db], xs[i].soff, xs[i].doff, xs[i].bytes);
            o += t;
        }
        return o + "]";
    };
    char head[512];
    snprintf(head, sizeof(head),
             "{\"G\": %d, \"g\": %d, \"m\": %d, \"mloc\": %d, \"K\": %d, \"n\": %llu, \"N\": %llu, \"Nloc\": %llu, "
             "\"buffers\": {\"A\": %zu, \"B\": %zu, \"W\": %zu, \"T\": %zu, \"X\": %zu, \"HALO\": %zu, "
             "\"COPY_A\": %zu, \"COPY_B\": %zu}, \"top_cross\": [",
             S.G, S.g, S.m, S.mloc, S.K, (unsigned long long)S.n, (unsigned long long)S.N, (unsigned long long)S.Nloc,
             S.off[SB_B] - S.off[SB_A], S.off[SB_W] - S.off[SB_B], S.off[SB_T] - S.off[SB_W], S.off[SB_X] - S.off[SB_T],
             S.off[SB_HALO] - S.off[SB_X], S.off[SB_CA] - S.off[SB_HALO], S.off[SB_CB] - S.off[SB_CA],
             S.bytes - S.off[SB_CB]);
    std::string out = head;
    for (size_t i = 0; i < S.top_cross.size(); i++) out += (i ? ", " : "") + std::to_string(S.top_cross[i]);
    out += "], \"gather\": " + list(X.gather) + ", \"xchg\": " + list(X.xchg);
    out += ", \"a2a_fwd\": " + list(X.a2a_fwd) + ", \"a2a_back\": " + list(X.a2a_back) + ", \"cross\": [";
    for (size_t i = 0; i < X.cross.size(); i++) out += (i ? ", " : "") + list(X.cross[i]);
    out += "], \"halo\": " + list(X.halo) + "}";
    if (buf && cap) {
        const size_t n = std::min(cap - 1, out.size());
        memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return (int)out.size() + 1;
}

gf2x_status gf2x_profile_enable(int on) {
    prof_clear();
    g_prof_on = on != 0;
    return GF2X_OK;
}

int gf2x_profile_report(char* buf, size_t cap) {
    // aggregate by kernel name, in first-seen order
    std::vector<std::string> order;
    std::map<std::string, std::pair<int, std::pair<double, double>>> agg;
    std::map<std::string, double> aops;
    for (auto& r : g_prof) {
        cudaEventSynchronize(r.end);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.beg, r.end);
        auto it = agg.find(r.name);
        if (it == agg.end()) {
            order.push_back(r.name);
            agg[r.name] = {0, {0.0, 0.0}};
        }
        auto& a = agg[r.name];
        a.first += r.launches;
        a.second.first += ms;
        a.second.second += r.bytes;
        aops[r.name] += r.ops;
    }
    std::string out = "[";
    for (size_t i = 0; i < order.size(); i++) {
        auto& a = agg[order[i]];
        char tmp[256];
        snprintf(tmp, sizeof(tmp), "%s{\"kernel\": \"%s\", \"launches\": %d, \"ms\": %.6f, \"bytes\": %.0f, \"alu_ops\": %.0f}",
                 i ? ", " : "", order[i].c_str(), a.first, a.second.first, a.second.second, aops[order[i]]);
        out += tmp;
    }
    out += "]";
    if (buf && cap) {
        size_t n = std::min(cap - 1, out.size());
        memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return (int)out.size() + 1;
}

const char* gf2x_status_string(gf2x_status s) {
    switch (s) {
        case GF2X_OK: return "ok";
        case GF2X_EINVAL: return "invalid argument";
        case GF2X_ETOOBIG: return "size too big";
        case GF2X_ENOMEM: return "out of memory";
        case GF2X_ECUDA: return "CUDA error";
        case GF2X_ENCCL: return "NCCL error";
    }
    return "unknown status";
}

const char* gf2x_last_error(void) { return g_last_error.c_str(); }

gf2x_status gf2x_release(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_dev.find(device);
    if (it == g_dev.end()) return GF2X_OK;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (auto& kv : it->second.ws)
        if (kv.second.first) cudaFree(kv.second.first);
    for (void* p : it->second.retired) cudaFree(p);
    if (it->second.tabs) cudaFree(it->second.tabs);
    if (it->second.shard_ws) cudaFree(it->second.shard_ws);
    if (it->second.tabs256) cudaFree(it->second.tabs256);
    if (it->second.tabsA4) cudaFree(it->second.tabsA4);
    for (auto& f : it->second.frob) cudaFree(f.second);
    delete it->second.host;
    g_dev.erase(it);
    cudaSetDevice(cur);
    return GF2X_OK;
}

const char* gf2x_version(void) { return "gf2x-b200 0.3 (sm_100a; Alg. 5 w=64 TGF(2^128) and w=128 TGF(2^256); Alg. 4 GF(2^128))"; }

}  // extern "C"

#ifdef SM_TRACE
// (SM_TRACE builds only: the phase timestamps of the last k_small launch, 16 CTAs x 16 points)
extern "C" int gf2x_debug_small_trace(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_sm_trace, sizeof(g_sm_trace)) == cudaSuccess ? 0 : 1;
}
#endif
