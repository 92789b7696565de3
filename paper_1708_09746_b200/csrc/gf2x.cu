// gf2x.cu -- sm_100a implementation of the C ABI in include/gf2x.h.
//
// Pipeline (Alg. 5), per product of n_a x n_b 64-bit words, N = 2^m points:
//   k_prep          Split: copy + mask words into the conversion scratch S (u64)
//   k_cvt_*         BasisCvt (Alg. 3 P:518-539 / Alg. 2) on 64-bit words, in place in S
//   k_fft<psi>      changeRepr (§4.3) fused into the first FFT_LCH pass (Alg. 1)
//   k_fft           remaining FFT_LCH layers (tiles of layers through shared memory)
//   k_pointmul      pointmul: bit-sliced TGF(2^128) Karatsuba
//   k_fft<inverse>  iFFT_LCH
//   k_cvt_*         iBasisCvt on 128-bit tower elements
//   k_ipsi_combine  changeRepr back + InterleavedCombine
// Every step runs in these kernels; the host only plans passes and enqueues launches.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
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
    uint32_t cloc[63 * 128]; // M4R-4 tables of the fixed low multiplier parts s_k(phi(j 2^(k+1))), k < 6
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

// =============================================================================================
// Basis conversion.  One Taylor step ("op") of Alg. 2 on segments of 2^lg units, h = 2^(lg-1),
// u = h >> K, d = h - u, is the sequential loop  for i = 2h-1 .. h: f[i-d] ^= f[i]  (R4).
// It splits into two dependency-free sweeps ("phase A": targets [h, h+u), "phase B": targets
// [u, h)), both f[t] ^= f[t+d]; forward runs A then B, the inverse (ascending loop) B then A.
// =============================================================================================
struct CvtOp {
    int lg, K;
};
#define MAX_TILE_OPS 48
struct CvtTileParams {
    void* data;
    uint64_t units_per_pair;  // 2^m
    uint64_t batch;
    int m, c, r_lo, R;        // tile bits [0,c) U [r_lo, r_lo+R)  (contiguous: c = 0, r_lo = 0)
    int nops, inverse;
    CvtOp ops[MAX_TILE_OPS];
};

template <typename T>
__device__ __forceinline__ T xor_t(T a, T b);
template <>
__device__ __forceinline__ uint64_t xor_t<uint64_t>(uint64_t a, uint64_t b) { return a ^ b; }
template <>
__device__ __forceinline__ uint4 xor_t<uint4>(uint4 a, uint4 b) { return xor4(a, b); }

// global index (within the pair) of tile slot s
__device__ __forceinline__ uint64_t tile_index(uint64_t base, uint64_t s, int c, int r_lo) {
    const uint64_t col = s & ((1ull << c) - 1), row = s >> c;
    return base | col | (row << r_lo);
}
__device__ __forceinline__ uint64_t tile_slot(uint64_t g, int c, int r_lo, int R) {
    return (g & ((1ull << c) - 1)) | (((g >> r_lo) & ((1ull << R) - 1)) << c);
}
// base index (within the pair) of tile t of a pair, tile bits [0,c) U [r_lo, r_lo+R)
__device__ __forceinline__ uint64_t tile_base(uint64_t t, int c, int r_lo, int R) {
    const int midbits = r_lo - c;
    const uint64_t mid = t & ((1ull << midbits) - 1), hi = t >> midbits;
    return (mid << c) | (hi << (r_lo + R));
}

template <typename T>
__device__ void cvt_sweep(T* tile, uint64_t base, int c, int r_lo, int R, int lg, int K, int phaseA) {
    const uint64_t h = 1ull << (lg - 1), u = h >> K, d = h - u;
    const uint64_t nslots = 1ull << (c + R);
    for (uint64_t s = threadIdx.x; s < nslots; s += blockDim.x) {
        const uint64_t g = tile_index(base, s, c, r_lo);
        const uint64_t pos = g & ((h << 1) - 1);
        const bool tgt = phaseA ? (pos >= h && pos < h + u) : (pos >= u && pos < h);
        if (tgt) {
            const uint64_t src = tile_slot(g + d, c, r_lo, R);
            tile[s] = xor_t<T>(tile[s], tile[src]);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_cvt_tile(CvtTileParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw);
    T* data = reinterpret_cast<T*>(p.data);
    const uint64_t nslots = 1ull << (p.c + p.R);
    const uint64_t tiles_per_pair = p.units_per_pair >> (p.c + p.R);
    const uint64_t ntiles = tiles_per_pair * p.batch;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t pair = t / tiles_per_pair, tt = t - pair * tiles_per_pair;
        const uint64_t base = tile_base(tt, p.c, p.r_lo, p.R);
        T* dp = data + pair * p.units_per_pair;
        for (uint64_t s = threadIdx.x; s < nslots; s += blockDim.x) tile[s] = dp[tile_index(base, s, p.c, p.r_lo)];
        __syncthreads();
        for (int o = 0; o < p.nops; o++) {
            const CvtOp op = p.ops[o];
            cvt_sweep<T>(tile, base, p.c, p.r_lo, p.R, op.lg, op.K, p.inverse ? 0 : 1);
            __syncthreads();
            cvt_sweep<T>(tile, base, p.c, p.r_lo, p.R, op.lg, op.K, p.inverse ? 1 : 0);
            __syncthreads();
        }
        for (uint64_t s = threadIdx.x; s < nslots; s += blockDim.x) dp[tile_index(base, s, p.c, p.r_lo)] = tile[s];
        __syncthreads();
    }
}

// One sweep of one op over the whole array (used when the op's window does not fit a tile).
template <typename T>
__global__ void k_cvt_stream(T* __restrict__ data, uint64_t total_units, int lg, int K, int phaseA) {
    const uint64_t h = 1ull << (lg - 1), u = h >> K, d = h - u;
    const uint64_t len = h << 1;
    // targets per segment: phase A -> u of them starting at h; phase B -> h-u starting at u
    const uint64_t per = phaseA ? u : (h - u);
    const uint64_t first = phaseA ? h : u;
    const uint64_t ntgt = (total_units / len) * per;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ntgt; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t seg = i / per, j = i - seg * per;
        const uint64_t t = seg * len + first + j;
        data[t] = xor_t<T>(data[t], data[t + d]);
    }
}

#include "fft.cuh"

// =============================================================================================
// pointmul: P[i] = A[i] (x) B[i] in TGF(2^128).  32 consecutive elements per thread are
// bit-sliced (transpose32), multiplied with the generated straight-line Karatsuba (bs_mul32 for the
// TGF(2^32) limb products, XOR networks for the fixed constants v31, v31^2), and transposed back.
//   a = alpha0 + alpha1 x7, alpha_i = A_2i + A_2i+1 x6 (limbs), x6^2 = x6 + v31, x7^2 = x7 + v63,
//   v63 = v31 x6  =>  v63 (e0 + e1 x6) = v31^2 e1 + v31 (e0 + e1) x6.
// =============================================================================================
#define PM_THREADS 64
#define PM_ROW 129   // 32 elements x 4 words + 1 pad word (conflict-free strided access)

__device__ __forceinline__ void load_planes(const uint32_t* rowA, int limb, uint32_t* x) {
#pragma unroll
    for (int e = 0; e < 32; e++) x[e] = rowA[e * 4 + limb];
    transpose32(x);
}
__device__ __forceinline__ void load_planes_sum(const uint32_t* row, int l0, int l1, uint32_t* x) {
#pragma unroll
    for (int e = 0; e < 32; e++) x[e] = row[e * 4 + l0] ^ row[e * 4 + l1];
    transpose32(x);
}

// TGF(2^64) product of bit-sliced (g0 + g1 x6)(d0 + d1 x6); operands given by loader lambdas
template <typename LA, typename LB>
__device__ __forceinline__ void bs_mul64(LA la, LB lb, uint32_t* r0, uint32_t* r1) {
    uint32_t x[32], y[32], p0[32], p2[32], t[32];
    la(0, x); lb(0, y);
    bs_mul32(x, y, p0);
    la(1, x); lb(1, y);
    bs_mul32(x, y, p2);
    la(2, x); lb(2, y);          // g0 + g1, d0 + d1
    bs_mul32(x, y, t);           // p1
#pragma unroll
    for (int i = 0; i < 32; i++) r1[i] = t[i] ^ p0[i];
    bs_mul_v31(p2, t);
#pragma unroll
    for (int i = 0; i < 32; i++) r0[i] = p0[i] ^ t[i];
}

__global__ void __launch_bounds__(PM_THREADS) k_pointmul(uint4* __restrict__ A, const uint4* __restrict__ B, uint64_t total) {
    extern __shared__ __align__(16) uint32_t pm_smem[];
    uint32_t* sa = pm_smem;                          // PM_THREADS rows of PM_ROW
    uint32_t* sb = sa + PM_THREADS * PM_ROW;
    uint32_t* scr = sb + PM_THREADS * PM_ROW;        // per thread 128 words
    const uint64_t per_cta = PM_THREADS * 32ull;
    const uint64_t ntiles = (total + per_cta - 1) / per_cta;
    uint32_t* rowA = sa + threadIdx.x * PM_ROW;
    uint32_t* rowB = sb + threadIdx.x * PM_ROW;
    uint32_t* my = scr + threadIdx.x * 128;
    for (uint64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        const uint64_t e0 = tl * per_cta;
        for (uint64_t i = threadIdx.x; i < per_cta; i += PM_THREADS) {
            const uint64_t e = e0 + i;
            uint4 va = make_uint4(0, 0, 0, 0), vb = make_uint4(0, 0, 0, 0);
            if (e < total) { va = A[e]; vb = B[e]; }
            uint32_t* ra = sa + (i >> 5) * PM_ROW + (i & 31) * 4;
            uint32_t* rb = sb + (i >> 5) * PM_ROW + (i & 31) * 4;
            ra[0] = va.x; ra[1] = va.y; ra[2] = va.z; ra[3] = va.w;
            rb[0] = vb.x; rb[1] = vb.y; rb[2] = vb.z; rb[3] = vb.w;
        }
        __syncthreads();
        uint32_t h0[32], h1[32];
        // q1 = (alpha0 + alpha1)(beta0 + beta1); limbs of alpha0+alpha1: (A0^A2, A1^A3), sum (A0^A1^A2^A3)
        {
            auto la = [&](int w, uint32_t* x) {
                if (w == 0) load_planes_sum(rowA, 0, 2, x);
                else if (w == 1) load_planes_sum(rowA, 1, 3, x);
                else {
#pragma unroll
                    for (int e = 0; e < 32; e++) x[e] = rowA[e * 4] ^ rowA[e * 4 + 1] ^ rowA[e * 4 + 2] ^ rowA[e * 4 + 3];
                    transpose32(x);
                }
            };
            auto lb = [&](int w, uint32_t* x) {
                if (w == 0) load_planes_sum(rowB, 0, 2, x);
                else if (w == 1) load_planes_sum(rowB, 1, 3, x);
                else {
#pragma unroll
                    for (int e = 0; e < 32; e++) x[e] = rowB[e * 4] ^ rowB[e * 4 + 1] ^ rowB[e * 4 + 2] ^ rowB[e * 4 + 3];
                    transpose32(x);
                }
            };
            bs_mul64(la, lb, h0, h1);
#pragma unroll
            for (int i = 0; i < 32; i++) { my[i] = h0[i]; my[32 + i] = h1[i]; }
        }
        // q0 = alpha0 beta0 ; hi = q1 + q0
        {
            auto la = [&](int w, uint32_t* x) { if (w < 2) load_planes(rowA, w, x); else load_planes_sum(rowA, 0, 1, x); };
            auto lb = [&](int w, uint32_t* x) { if (w < 2) load_planes(rowB, w, x); else load_planes_sum(rowB, 0, 1, x); };
            bs_mul64(la, lb, h0, h1);
#pragma unroll
            for (int i = 0; i < 32; i++) {
                my[i] ^= h0[i]; my[32 + i] ^= h1[i];      // hi
                my[64 + i] = h0[i]; my[96 + i] = h1[i];  // q0
            }
        }
        // q2 = alpha1 beta1 ; lo = q0 + v63 q2
        {
            auto la = [&](int w, uint32_t* x) { if (w < 2) load_planes(rowA, 2 + w, x); else load_planes_sum(rowA, 2, 3, x); };
            auto lb = [&](int w, uint32_t* x) { if (w < 2) load_planes(rowB, 2 + w, x); else load_planes_sum(rowB, 2, 3, x); };
            bs_mul64(la, lb, h0, h1);   // q2 = (e0, e1)
            uint32_t t[32], u[32];
            // v63 (e0 + e1 x6) = v31^2 e1 + v31 (e0 + e1) x6
            bs_mul_v31sq(h1, t);
#pragma unroll
            for (int i = 0; i < 32; i++) u[i] = h0[i] ^ h1[i];
            bs_mul_v31(u, h1);
#pragma unroll
            for (int i = 0; i < 32; i++) {
                h0[i] = my[64 + i] ^ t[i];   // lo limb 0
                h1[i] ^= my[96 + i];         // lo limb 1
            }
        }
        // write back: result limbs (lo0, lo1, hi0, hi1) -> transpose -> rowA
        __syncwarp();
        transpose32(h0);
#pragma unroll
        for (int e = 0; e < 32; e++) rowA[e * 4 + 0] = h0[e];
        transpose32(h1);
#pragma unroll
        for (int e = 0; e < 32; e++) rowA[e * 4 + 1] = h1[e];
#pragma unroll
        for (int i = 0; i < 32; i++) h0[i] = my[i];
        transpose32(h0);
#pragma unroll
        for (int e = 0; e < 32; e++) rowA[e * 4 + 2] = h0[e];
#pragma unroll
        for (int i = 0; i < 32; i++) h1[i] = my[32 + i];
        transpose32(h1);
#pragma unroll
        for (int e = 0; e < 32; e++) rowA[e * 4 + 3] = h1[e];
        __syncthreads();
        for (uint64_t i = threadIdx.x; i < per_cta; i += PM_THREADS) {
            const uint64_t e = e0 + i;
            if (e < total) {
                const uint32_t* ra = sa + (i >> 5) * PM_ROW + (i & 31) * 4;
                A[e] = make_uint4(ra[0], ra[1], ra[2], ra[3]);
            }
        }
        __syncthreads();
    }
}

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

__global__ void __launch_bounds__(256) k_ipsi_combine(const uint4* __restrict__ P, const DevTables* tabs, uint64_t N,
                                                      uint64_t n_out, uint64_t batch, uint64_t* __restrict__ out) {
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
                if (w >= 1 && w - 1 < N) {
                    uint64_t l2;
                    ipsi_apply(itab, P[pair * N + w - 1], l2, prev_hi);
                }
            }
            out[i] = lo ^ prev_hi;
        }
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
    double bytes;
};
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
    ProfScope(const char* name, double bytes, cudaStream_t s) : st(s) {
        if (!g_prof_on) return;
        ProfRec r{name, prof_event(), prof_event(), bytes};
        cudaEventRecord(r.beg, st);
        g_prof.push_back(r);
        idx = (int)g_prof.size() - 1;
    }
    ~ProfScope() {
        if (idx >= 0) cudaEventRecord(g_prof[idx].end, st);
    }
};

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
    int sm_count = 0;
    std::map<cudaStream_t, std::pair<void*, size_t>> ws;  // per-stream workspace cache
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
    // cloc: fixed low parts for the bottom FFT pass: table id 2^(BOT_B-1-k) - 1 + j holds the
    // constant s_k(phi(j 2^(k+1))) (local index bits (k, BOT_B)), k < BOT_B
    for (int k = 0; k < BOT_B; k++)
        for (int j = 0; j < (1 << (BOT_B - 1 - k)); j++) {
            uint32_t bb = (uint32_t)j << (k + 1), e = 0;
            for (int i = k + 1; i < BOT_B; i++)
                if ((bb >> i) & 1) e ^= T->S[k * 32 + i];
            uint32_t* tab = T->cloc + (((1 << (BOT_B - 1 - k)) - 1) + j) * 128;
            for (int t = 0; t < 8; t++)
                for (int x = 0; x < 16; x++) tab[16 * t + x] = (uint32_t)tower_mul((u128)e, ((u128)x) << (4 * t));
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
        delete h;
        if (e != cudaSuccess) { cudaFree(d); return fail(GF2X_ECUDA, cudaGetErrorString(e)); }
        CUDA_TRY(cudaDeviceGetAttribute(&st.sm_count, cudaDevAttrMultiProcessorCount, dev));
        // opt-in shared memory sizes
        CUDA_TRY(cudaFuncSetAttribute(k_fft2<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft2<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft2<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft2<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft2<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft2<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_tile<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_cvt_tile<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_pointmul, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_ipsi_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
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

// BasisCvt schedule (Alg. 3 with the paper's largest-K split, R4-R6) as global ops
static void cvt_ops(int m, int sigma, std::vector<CvtOp>& out) {
    if (m <= 1) return;
    int K = 1;
    while (2 * K <= m - 1) K *= 2;
    for (int l = m; l >= K + 1; --l) out.push_back({l + sigma, K});
    cvt_ops(m - K, sigma + K, out);
    cvt_ops(K, sigma, out);
}

struct CvtPass {
    bool stream;
    int c, r_lo, R;          // tile passes
    std::vector<CvtOp> ops;  // tile: ops in execution order; stream: 1 op
};

// group ops into tile passes (windows [lg-1-K, lg) inside the tile bits) or streaming ops
static std::vector<CvtPass> plan_cvt(int m, int unit_bytes) {
    std::vector<CvtOp> ops;
    cvt_ops(m, 0, ops);
    const int T = (unit_bytes == 8) ? 13 : 12;     // 64 KB tiles
    const int cc = (unit_bytes == 8) ? 4 : 3;      // 128 B contiguous per row
    const int R = T - cc;
    std::vector<CvtPass> passes;
    for (const CvtOp& op : ops) {
        const int wlo = op.lg - 1 - op.K, whi = op.lg;
        if (!passes.empty() && !passes.back().stream && (int)passes.back().ops.size() < MAX_TILE_OPS) {
            CvtPass& P = passes.back();
            bool fits = (P.c == 0) ? (whi <= P.R) : (wlo >= P.r_lo && whi <= P.r_lo + P.R);
            if (fits) { P.ops.push_back(op); continue; }
        }
        CvtPass P;
        if (whi <= std::min(T, m)) {
            P.stream = false; P.c = 0; P.r_lo = 0; P.R = std::min(T, m);
        } else if (whi - wlo <= R && wlo >= cc) {
            P.stream = false; P.c = cc; P.R = R; P.r_lo = std::max(cc, whi - R);
            if (P.r_lo + P.R > m) P.r_lo = m - P.R;
            if (P.r_lo < cc) { P.stream = true; }
        } else {
            P.stream = true;
        }
        if (P.stream) { P.c = P.r_lo = P.R = 0; }
        P.ops.push_back(op);
        passes.push_back(P);
    }
    return passes;
}

struct FftPass {
    int c, k_lo, k_hi;  // direct: tile bits [0,c) U [k_lo,k_hi); bottom: c = k_lo = 0, k_hi = Rt
    bool bottom;
    int layers;         // bottom: layers [0, layers)
};
// forward order (top-down); the first pass also applies changeRepr.  High layers [BOT_B, m) are
// split evenly into direct passes of <= 6 layers; layers [0, min(m, BOT_B)) form the bottom pass.
static std::vector<FftPass> plan_fft(int m) {
    std::vector<FftPass> v;
    const int H = m > BOT_B ? m - BOT_B : 0;
    const int np = (H + 5) / 6;
    int top = m;
    for (int i = 0; i < np; i++) {
        const int rem = top - BOT_B;
        const int r = (rem + (np - i) - 1) / (np - i);  // remaining layers / remaining passes
        const int lo = top - r;
        v.push_back({i == 0 ? 5 : 6, lo, top, false, 0});
        top = lo;
    }
    const int rt = m < BOT_RT ? m : BOT_RT;
    v.push_back({0, 0, rt, true, m < BOT_B ? m : BOT_B});
    return v;
}

struct Plan {
    uint64_t na, nb, N, batch;
    int m, ma, mb;
    std::vector<CvtPass> cvt_a, cvt_b, icvt;
    std::vector<FftPass> fft;
    size_t off_sa, off_sb, off_wa, off_wb, bytes;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static gf2x_status make_plan(uint64_t a_bits, uint64_t b_bits, int64_t batch, Plan& P) {
    if (batch < 0) return fail(GF2X_EINVAL, "negative batch");
    P.na = (a_bits + 63) / 64;
    P.nb = (b_bits + 63) / 64;
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
    P.fft = plan_fft(P.m);
    const uint64_t spec = P.N * P.batch + 2048;  // pad for the pointmul tile
    P.off_sa = 0;
    P.off_sb = align256(P.off_sa + (1ull << P.ma) * P.batch * 8);
    P.off_wa = align256(P.off_sb + (1ull << P.mb) * P.batch * 8);
    P.off_wb = align256(P.off_wa + spec * 16);
    P.bytes = align256(P.off_wb + spec * 16);
    return GF2X_OK;
}

static int launches_of(const Plan& P) {
    int n = 2;  // prep a, b
    for (auto* v : {&P.cvt_a, &P.cvt_b, &P.icvt})
        for (auto& p : *v) n += p.stream ? 2 : 1;
    n += 2 * (int)P.fft.size();  // forward a, b
    n += 1;                      // pointmul
    n += (int)P.fft.size();      // inverse
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

template <typename T>
static gf2x_status run_cvt(const std::vector<CvtPass>& passes, T* data, int m, uint64_t batch, bool inverse,
                           int sm_count, cudaStream_t st) {
    const uint64_t per = 1ull << m;
    std::vector<const CvtPass*> order;
    for (auto& p : passes) order.push_back(&p);
    if (inverse) std::reverse(order.begin(), order.end());
    for (const CvtPass* pp : order) {
        const CvtPass& p = *pp;
        if (p.stream) {
            const CvtOp op = p.ops[0];
            const uint64_t h = 1ull << (op.lg - 1), u = h >> op.K;
            const uint64_t nA = (per * batch >> op.lg) * u, nB = (per * batch >> op.lg) * (h - u);
            const int first = inverse ? 0 : 1;  // phaseA flag of the first sweep
            for (int sw = 0; sw < 2; sw++) {
                const int phaseA = (sw == 0) ? first : 1 - first;
                const uint64_t n = phaseA ? nA : nB;
                ProfScope ps(sizeof(T) == 8 ? "k_cvt_stream<u64>" : "k_cvt_stream<u128>", 3.0 * n * sizeof(T), st);
                k_cvt_stream<T><<<grid_for(n, 256, sm_count, 8), 256, 0, st>>>(data, per * batch, op.lg, op.K, phaseA);
            }
        } else {
            CvtTileParams prm;
            prm.data = data;
            prm.units_per_pair = per;
            prm.batch = batch;
            prm.m = m; prm.c = p.c; prm.r_lo = p.r_lo; prm.R = p.R;
            prm.inverse = inverse ? 1 : 0;
            prm.nops = (int)p.ops.size();
            for (int i = 0; i < prm.nops; i++) prm.ops[i] = inverse ? p.ops[prm.nops - 1 - i] : p.ops[i];
            const size_t sm = ((size_t)1 << (p.c + p.R)) * sizeof(T);
            const uint64_t ntiles = (per >> (p.c + p.R)) * batch;
            ProfScope ps(sizeof(T) == 8 ? "k_cvt_tile<u64>" : "k_cvt_tile<u128>", 2.0 * per * batch * sizeof(T), st);
            k_cvt_tile<T><<<grid_for(ntiles, 1, sm_count, 3), 256, sm, st>>>(prm);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("cvt launch: ") + cudaGetErrorString(e));
    }
    return GF2X_OK;
}

static gf2x_status launch_fft(const FftPass& f, bool inv, bool psi, const void* src, uint64_t src_per, uint4* dst,
                              const Plan& P, DeviceState* ds, cudaStream_t st) {
    FftParams prm;
    prm.src = src; prm.dst = dst; prm.tabs = ds->tabs;
    prm.src_per = src_per; prm.batch = P.batch;
    prm.m = P.m; prm.c = f.c; prm.k_lo = f.k_lo; prm.k_hi = f.k_hi; prm.layers = f.layers;
    const int R = f.k_hi - f.k_lo;
    const uint64_t ntiles = (P.N >> (f.c + R)) * P.batch;
    const size_t sm = fft2_smem(f.c, R, f.layers, psi, f.bottom);
    const int occ = sm > 113 * 1024 ? 1 : (sm > 75 * 1024 ? 2 : 3);
    const int grid = grid_for(ntiles, 1, ds->sm_count, occ);
    const double bytes = (double)P.batch * (psi ? (double)src_per * 8 : (double)P.N * 16) + (double)P.batch * P.N * 16;
    ProfScope ps(f.bottom ? (inv ? "k_fft_bottom<inv>" : (psi ? "k_fft_bottom<psi>" : "k_fft_bottom"))
                          : (inv ? "k_fft<inv>" : (psi ? "k_fft<psi>" : "k_fft")), bytes, st);
    if (f.bottom) {
        if (inv) k_fft2<true, false, true><<<grid, FFT_THREADS, sm, st>>>(prm);
        else if (psi) k_fft2<false, true, true><<<grid, FFT_THREADS, sm, st>>>(prm);
        else k_fft2<false, false, true><<<grid, FFT_THREADS, sm, st>>>(prm);
    } else {
        if (inv) k_fft2<true, false, false><<<grid, FFT_THREADS, sm, st>>>(prm);
        else if (psi) k_fft2<false, true, false><<<grid, FFT_THREADS, sm, st>>>(prm);
        else k_fft2<false, false, false><<<grid, FFT_THREADS, sm, st>>>(prm);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("fft launch: ") + cudaGetErrorString(e));
    return GF2X_OK;
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
    // Split
    {
        ProfScope ps("k_prep", (double)P.batch * (P.na + (1ull << P.ma)) * 8, st);
        k_prep<<<grid_for((1ull << P.ma) * P.batch, 256, smc, 8), 256, 0, st>>>(a, P.na, a_bits, P.ma, P.batch, Sa);
    }
    {
        ProfScope ps("k_prep", (double)P.batch * (P.nb + (1ull << P.mb)) * 8, st);
        k_prep<<<grid_for((1ull << P.mb) * P.batch, 256, smc, 8), 256, 0, st>>>(b, P.nb, b_bits, P.mb, P.batch, Sb);
    }
    // BasisCvt on 64-bit blocks
    if ((s = run_cvt<uint64_t>(P.cvt_a, Sa, P.ma, P.batch, false, smc, st)) != GF2X_OK) return s;
    if ((s = run_cvt<uint64_t>(P.cvt_b, Sb, P.mb, P.batch, false, smc, st)) != GF2X_OK) return s;
    // changeRepr + FFT_LCH
    for (size_t i = 0; i < P.fft.size(); i++) {
        const bool first = (i == 0);
        const bool only_psi = (stop_stage == 1);
        FftPass f = P.fft[i];
        if (only_psi) {  // changeRepr only
            if (!first) break;
            if (f.bottom) f.layers = 0; else f.k_lo = f.k_hi;
        }
        if ((s = launch_fft(f, false, first, first ? (const void*)Sa : Wa, first ? (1ull << P.ma) : P.N, Wa, P, ds, st)) != GF2X_OK) return s;
        if ((s = launch_fft(f, false, first, first ? (const void*)Sb : Wb, first ? (1ull << P.mb) : P.N, Wb, P, ds, st)) != GF2X_OK) return s;
    }
    if (stop_stage == 1 || stop_stage == 2) return GF2X_OK;
    // pointmul
    {
        const uint64_t total = P.N * P.batch;
        const uint64_t ntiles = (total + PM_THREADS * 32 - 1) / (PM_THREADS * 32);
        const size_t sm = (size_t)(2 * PM_THREADS * PM_ROW + PM_THREADS * 128) * 4;
        ProfScope ps("k_pointmul", 48.0 * total, st);
        k_pointmul<<<grid_for(ntiles, 1, smc, 2), PM_THREADS, sm, st>>>(Wa, Wb, total);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string("pointmul launch: ") + cudaGetErrorString(e));
    }
    if (stop_stage == 3) return GF2X_OK;
    // iFFT_LCH (passes in reverse order)
    for (size_t i = P.fft.size(); i-- > 0;) {
        if ((s = launch_fft(P.fft[i], true, false, Wa, P.N, Wa, P, ds, st)) != GF2X_OK) return s;
    }
    if (stop_stage == 4) return GF2X_OK;
    // iBasisCvt (tower)
    if ((s = run_cvt<uint4>(P.icvt, Wa, P.m, P.batch, true, smc, st)) != GF2X_OK) return s;
    if (stop_stage == 5) return GF2X_OK;
    // changeRepr^-1 + InterleavedCombine
    {
        const uint64_t n_out = P.na + P.nb;
        const uint64_t total = n_out * P.batch;
        ProfScope ps("k_ipsi_combine", 16.0 * P.N * P.batch + 8.0 * total, st);
        k_ipsi_combine<<<grid_for(total, 256, smc, 2), 256, 16 * 256 * 16, st>>>(Wa, ds->tabs, P.N, n_out, P.batch, c);
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

static gf2x_status mul_common(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                              int64_t batch, void* user_ws, size_t user_ws_bytes, void* stream, int stop_stage,
                              uint64_t* stage_out) {
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
    void* ws = user_ws;
    if (ws) {
        if (user_ws_bytes < P.bytes) return fail(GF2X_ENOMEM, "workspace too small");
    } else {
        std::lock_guard<std::mutex> lk(g_mu);
        auto& ent = ds->ws[st];
        if (ent.second < P.bytes) {
            if (ent.first) {
                cudaStreamSynchronize(st);
                cudaFree(ent.first);
                ent.first = nullptr;
                ent.second = 0;
            }
            void* p = nullptr;
            cudaError_t e = cudaMalloc(&p, P.bytes);
            if (e != cudaSuccess) return fail(GF2X_ENOMEM, std::string("workspace: ") + cudaGetErrorString(e));
            ent.first = p;
            ent.second = P.bytes;
        }
        ws = ent.first;
    }
    s = run_pipeline(a, a_bits, b, b_bits, c, P, ws, ds, st, stop_stage);
    if (s != GF2X_OK) return s;
    if (stop_stage && stage_out) {
        CUDA_TRY(cudaMemcpyAsync(stage_out, reinterpret_cast<unsigned char*>(ws) + P.off_wa, P.N * 16,
                                 cudaMemcpyDeviceToDevice, st));
    }
    return GF2X_OK;
}

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
    return launches_of(P);
}

gf2x_status gf2x_debug_stage(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, int stage,
                             uint64_t* out, void* stream) {
    if (stage < 1 || stage > 5 || !out || a_bits == 0 || b_bits == 0) return fail(GF2X_EINVAL, "bad debug stage request");
    return mul_common(a, a_bits, b, b_bits, nullptr, 1, nullptr, 0, stream, stage, out);
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
        a.first += 1;
        a.second.first += ms;
        a.second.second += r.bytes;
    }
    std::string out = "[";
    for (size_t i = 0; i < order.size(); i++) {
        auto& a = agg[order[i]];
        char tmp[256];
        snprintf(tmp, sizeof(tmp), "%s{\"kernel\": \"%s\", \"launches\": %d, \"ms\": %.6f, \"bytes\": %.0f}",
                 i ? ", " : "", order[i].c_str(), a.first, a.second.first, a.second.second);
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
    if (it->second.tabs) cudaFree(it->second.tabs);
    g_dev.erase(it);
    cudaSetDevice(cur);
    return GF2X_OK;
}

const char* gf2x_version(void) { return "gf2x-b200 0.1 (sm_100a, Alg. 5 TGF(2^128))"; }

}  // extern "C"
