// cvt.cuh -- BasisCvt / iBasisCvt kernels (Alg. 3 P:518-539 with VarSubs = Alg. 2),
// included by gf2x.cu.  XOR only; the same code converts 64-bit blocks (forward, before
// changeRepr) and 128-bit tower elements (inverse).
//
// One Taylor step ("op") of Alg. 2 on segments of 2^lg units, h = 2^(lg-1), u = h >> K, d = h - u,
// is the sequential loop  for i = 2h-1 .. h: f[i-d] ^= f[i]  (R4).  In the coordinate
// y = (i mod 2^lg) / u of its index window [lg-1-K, lg) it reads
//     phase A:  f[tau] ^= f[2 tau - 1]                    (tau = 2^K)
//     phase B:  f[y]   ^= f[y + tau - 1],  y = 1 .. tau-1
// and the two phases are dependency-free sweeps; the inverse (ascending loop) runs B then A.
#pragma once

struct CvtOp {
    int lg, K;
};
#define MAX_TILE_OPS 64
struct CvtTileParams {
    void* data;
    uint64_t units_per_pair;  // 2^m
    uint64_t batch;
    int c, r_lo, R;           // tile bits [0,c) U [r_lo, r_lo+R); op windows lie inside [r_lo, r_lo+R)
    int nops, inverse;
    CvtOp ops[MAX_TILE_OPS];
};

template <typename T>
__device__ __forceinline__ T xor_t(T a, T b);
template <>
__device__ __forceinline__ uint64_t xor_t<uint64_t>(uint64_t a, uint64_t b) { return a ^ b; }
template <>
__device__ __forceinline__ uint4 xor_t<uint4>(uint4 a, uint4 b) { return xor4(a, b); }

template <typename T>
__device__ __forceinline__ void cvt_phase(T* tile, uint32_t nslots, int sw0, int K, bool phaseA) {
    const uint32_t tau = 1u << K;
    const uint32_t lowm = (1u << sw0) - 1;
    if (phaseA) {
        const uint32_t nlines = nslots >> (K + 1);
        for (uint32_t ln = threadIdx.x; ln < nlines; ln += blockDim.x) {
            const uint32_t dep = (ln & lowm) | ((ln >> sw0) << (sw0 + K + 1));
            const uint32_t t = dep | (tau << sw0), src = dep | ((2 * tau - 1) << sw0);
            tile[t] = xor_t<T>(tile[t], tile[src]);
        }
    } else {
        // enumerate the slots whose top window bit is 0 with the lowest slot bits fastest, so that
        // consecutive lanes touch consecutive units (bank-conflict free); y = 0 does nothing
        const uint32_t n = nslots >> 1;
        const int tb = sw0 + K;                        // slot bit of the window's top bit
        const uint32_t off = (tau - 1) << sw0;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t y = (i >> sw0) & (tau - 1);
            if (!y) continue;
            const uint32_t t = (i & ((1u << tb) - 1)) | ((i >> tb) << (tb + 1));
            tile[t] = xor_t<T>(tile[t], tile[t + off]);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(512) k_cvt_tile(CvtTileParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw);
    T* data = reinterpret_cast<T*>(p.data);
    const uint32_t nslots = 1u << (p.c + p.R);
    const uint32_t cmask = (1u << p.c) - 1;
    const uint64_t tiles_per_pair = p.units_per_pair >> (p.c + p.R);
    const uint64_t ntiles = tiles_per_pair * p.batch;
    const int midbits = p.r_lo - p.c;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t pair = t / tiles_per_pair;
        const uint64_t tt = t - pair * tiles_per_pair;
        const uint64_t base = ((tt & ((1ull << midbits) - 1)) << p.c) | ((tt >> midbits) << (p.r_lo + p.R));
        T* dp = data + pair * p.units_per_pair + base;
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x)
            tile[s] = dp[(uint64_t)(s & cmask) | ((uint64_t)(s >> p.c) << p.r_lo)];
        __syncthreads();
        for (int o = 0; o < p.nops; o++) {
            const CvtOp op = p.ops[o];
            const int sw0 = p.c + (op.lg - 1 - op.K) - p.r_lo;   // slot bit of the window start
            cvt_phase<T>(tile, nslots, sw0, op.K, !p.inverse);
            __syncthreads();
            cvt_phase<T>(tile, nslots, sw0, op.K, p.inverse != 0);
            __syncthreads();
        }
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x)
            dp[(uint64_t)(s & cmask) | ((uint64_t)(s >> p.c) << p.r_lo)] = tile[s];
        __syncthreads();
    }
}

// One op over the whole array (its window does not fit a tile), both phases in one launch:
// the thread of phase-B target t in [u, 2u) also owns the phase-A target t + d (which only it reads).
template <typename T>
__global__ void __launch_bounds__(256) k_cvt_stream(T* __restrict__ data, uint64_t total_units, int lg, int K, int inverse) {
    const uint64_t h = 1ull << (lg - 1), u = h >> K, d = h - u;
    const uint64_t n = total_units >> 1;  // h slots per segment of 2h, j < u idle
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = i & (h - 1);
        if (j < u) continue;
        const uint64_t t = ((i >> (lg - 1)) << lg) + j;
        if (j < 2 * u) {
            const uint64_t tp = t + d;
            if (!inverse) {
                const T a = xor_t<T>(data[tp], data[tp + d]);
                data[tp] = a;
                data[t] = xor_t<T>(data[t], a);
            } else {
                data[t] = xor_t<T>(data[t], data[tp]);
                data[tp] = xor_t<T>(data[tp], data[tp + d]);
            }
        } else {
            data[t] = xor_t<T>(data[t], data[t + d]);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Residue-class pass: a run of Taylor steps with one K (levels lg_hi .. lg_lo, forward order) whose
// windows are wider than a tile.  Step lg couples f[i] with f[i + d], d = 2^(lg-1-K) (2^K - 1), so
// every step of the run maps each residue class i mod M, M = 2^K - 1, of a 2^q-unit chunk
// (q = lg_hi) to itself: with i = r M + c the class c is a column of rows r, and step lg is
// "row r ^= row r + u" (u = 2^(lg-1-K)) on the rows whose position i mod 2^lg lies in [u, h).
// A tile holds all rows of 2^C_log consecutive classes, so the whole run is one HBM pass instead
// of one streaming pass per step.  The target at position [u, 2u) also owns the phase-A target
// (position [h, h+u), row r + u) it reads, as in k_cvt_stream, so each step is one sweep.
// ---------------------------------------------------------------------------------------------
struct CvtResParams {
    void* data;
    uint64_t units_per_pair;  // 2^m
    uint64_t batch;
    int q, K, lg_hi, lg_lo, inverse;
    int C_log, rows;          // 2^C_log classes per tile; rows = floor((2^q - 1) / M) + 1
};

#define RES_THREADS 256
#define RES_MAXJ 18   // row slots per thread: rows <= RES_MAXJ * (RES_THREADS >> C_log) (checked by the planner)
#ifndef RES_UNROLL128
#define RES_UNROLL128 1   // measured: 128-bit units faster unrolled over 10 slots than rolled
#endif
// unrolled row slots: 64-bit units (C <= 32 classes: <= 18 slots); 128-bit units use C = 8 (<= 9 slots)
#define RES_SLOTS128 10
#define RES_SLOTS(T) ((sizeof(T) == 8 || !RES_UNROLL128) ? RES_MAXJ : RES_SLOTS128)
template <typename T>
__device__ __forceinline__ void cp_async_unit(T* dst, const T* src) {
    if (sizeof(T) == 16) cp_async16(dst, src);
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Thread (column c = tid mod C, row lane rl = tid / C) owns rows rl, rl + RS, ... (RS = threads / C) of
// its class; double-buffered: the next tile's rows are prefetched with cp.async during the steps.
template <typename T>
__device__ __forceinline__ void cvt_res_tiles(const CvtResParams& p, T* data, uint64_t t_first, uint64_t t_step,
                                              unsigned char* smem_raw) {
    const uint32_t M = (1u << p.K) - 1;
    const uint32_t C = 1u << p.C_log;
    const uint32_t nrb = (M + C - 1) >> p.C_log;
    const uint32_t span = 1u << p.q;                       // q <= 31
    const uint64_t chunks = (p.units_per_pair >> p.q) * p.batch;
    const uint64_t ntiles = chunks * nrb;
    const uint32_t nslots = (uint32_t)p.rows << p.C_log;
    const uint32_t bufsz = (nslots * (uint32_t)sizeof(T) + 127) & ~127u;
    const int nsteps = p.lg_hi - p.lg_lo + 1;
    const uint32_t c = threadIdx.x & (C - 1), rl = threadIdx.x >> p.C_log, RS = blockDim.x >> p.C_log;
    auto geom = [&](uint64_t t, T*& dp, uint32_t& c0, uint32_t& cn) {
        const uint64_t chunk = t / nrb;
        c0 = (uint32_t)(t - chunk * nrb) << p.C_log;
        cn = min(C, M - c0);
        dp = data + chunk * span;
    };
    auto prefetch = [&](uint64_t t, T* buf) {
        T* dp; uint32_t c0, cn;
        geom(t, dp, c0, cn);
        if (c < cn)
            for (uint32_t r = rl; r < (uint32_t)p.rows; r += RS) {
                const uint32_t i = r * M + c0 + c;
                if (i < span) cp_async_unit<T>(buf + ((r << p.C_log) | c), dp + i);
            }
    };
    if (t_first < ntiles) prefetch(t_first, reinterpret_cast<T*>(smem_raw));
    cp_async_commit();
    int k = 0;
    for (uint64_t t = t_first; t < ntiles; t += t_step, k++) {
        if (t + t_step < ntiles) prefetch(t + t_step, reinterpret_cast<T*>(smem_raw + ((k + 1) & 1) * bufsz));
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        T* tile = reinterpret_cast<T*>(smem_raw + (k & 1) * bufsz);
        T* dp; uint32_t c0, cn;
        geom(t, dp, c0, cn);
        const bool colok = c < cn;
        // unit index of the thread's row slot j (r = rl + j RS), 0 if the slot is empty (position 0 is never a
        // target); the slot's tile index is s0 + j RES_THREADS (RS 2^C_log = blockDim = RES_THREADS)
        uint32_t ii[RES_MAXJ];
#pragma unroll
        for (int j = 0; j < RES_SLOTS(T); j++) {
            const uint32_t r = rl + j * RS;
            const uint32_t i = r * M + c0 + c;
            ii[j] = (colok && r < (uint32_t)p.rows && i < span) ? i : 0u;
        }
        const uint32_t s0 = (rl << p.C_log) | c;
        for (int o = 0; o < nsteps; o++) {
            const int lg = p.inverse ? p.lg_lo + o : p.lg_hi - o;
            const uint32_t h = 1u << (lg - 1), u = h >> p.K, segm = (2u << (lg - 1)) - 1;
            const uint32_t off = u << p.C_log;
            // branch-light: targets are the positions [u, h); the thread of a target at [u, 2u) also owns the
            // phase-A target s + off (position [h, h + u)), whose source is s + 2 off
            // (measured: the single-load form below is faster for 128-bit units, the two-branch form for 64-bit)
            auto slot = [&](uint32_t i, uint32_t s) {
                const uint32_t pos = i & segm;
                if (sizeof(T) == 16) {
                    const bool act = (pos - u) < (h - u);
                    const bool isA = pos < 2 * u;
                    if (act) {
                        T src = tile[s + off];
                        if (isA) {
                            const T a = xor_t<T>(src, tile[s + 2 * off]);
                            tile[s + off] = a;
                            if (!p.inverse) src = a;
                        }
                        tile[s] = xor_t<T>(tile[s], src);
                    }
                } else {
                    if (pos - u >= h - u) return;
                    if (pos < 2 * u) {
                        if (!p.inverse) {
                            const T a = xor_t<T>(tile[s + off], tile[s + 2 * off]);
                            tile[s + off] = a;
                            tile[s] = xor_t<T>(tile[s], a);
                        } else {
                            const T a = tile[s + off];
                            tile[s] = xor_t<T>(tile[s], a);
                            tile[s + off] = xor_t<T>(a, tile[s + 2 * off]);
                        }
                    } else {
                        tile[s] = xor_t<T>(tile[s], tile[s + off]);
                    }
                }
            };
#pragma unroll
            for (int j = 0; j < RES_SLOTS(T); j++) slot(ii[j], s0 + j * RES_THREADS);
            __syncthreads();
        }
        if (colok)
            for (uint32_t r = rl; r < (uint32_t)p.rows; r += RS) {
                const uint32_t i = r * M + c0 + c;
                if (i < span) dp[i] = tile[(r << p.C_log) | c];
            }
        __syncthreads();
    }
    cp_async_wait<0>();
}

template <typename T>
__global__ void __launch_bounds__(RES_THREADS, 3) k_cvt_res(CvtResParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    cvt_res_tiles<T>(p, reinterpret_cast<T*>(p.data), blockIdx.x, gridDim.x, smem_raw);
}

// ---------------------------------------------------------------------------------------------
// Seam pass (k_cvt_seam): a COMPLETE Taylor run (levels q .. K+1 of 2^q-unit chunks, Alg. 3 l.531 with
// Alg. 2's steps) in its closed form, R27.  With M = 2^K - 1, B = q - K and the
// residue classes c = 1 .. M (unit i = r M + c, row r; class M holds the units r M + M, i.e. the
// nonzero multiples of M; unit 0 is never a target), the run maps class c's rows x to
//     y[r] = XOR_{s superset of r} x[s]            for r <  c   (the superset-sum over the row bits)
//     y[r] = XOR_{s superset of r-1} x[s+1]        for r >= c   (the same transform of the rows shifted by one)
// (rows s run over 0 .. 2^B; a row beyond the chunk reads as 0).  For the classes c > 2^B of the top run
// (all but the first 2^B) only the first line applies: that is k_cvt_top's "generic" case (R24).
// Writing the class as (L = rows < c, U = rows >= c) and S = the superset-sum, the inverse run is
//     x_U = T y_U (T = the shifted transform, an involution on U),  v = S(x_U on U, 0 on L),
//     x_L = S(y_L on L, v on U) restricted to L                       (S_LL^-1 = S_LL, S_LL S_LU = S_LU S_UU).
// Each S is separable over the row bits, so a tile (all 2^B + 1 rows of 32 / W consecutive classes, W 32-bit
// words per unit: one 128-byte row, lane = word column) runs it in register phases of 4 row bits:
// forward 2 phases (low bits of P = S x and Q = T x, then the high bits and the seam select), inverse 4.
// Against k_cvt_res (one shared-memory sweep with a position test per step): the same HBM traffic and
// 2-4 register phases instead of 2 (q - K) sweeps.  B in [5, 8] (rows <= 257).
// ---------------------------------------------------------------------------------------------
#define SEAM_THREADS 256   // 2 CTAs per SM, one tile prefetched each (measured: 5 stages at one 512-thread CTA per
#define SEAM_NW (SEAM_THREADS / 32)   // SM 12 % slower; phase outputs stored straight to HBM 1.5x slower at u128)

template <int N>
__device__ __forceinline__ void seam_ss(uint32_t* v) {   // superset-sum over the log2(N) index bits
#pragma unroll
    for (int b = 1; b < N; b <<= 1)
#pragma unroll
        for (int t = 0; t < N; t++)
            if (!(t & b)) v[t] ^= v[t | b];
}

template <typename T>
__device__ __forceinline__ void seam_load_unit(T* dst, const T* src, bool ok) {
    const uint32_t n = ok ? (uint32_t)sizeof(T) : 0u;   // src-size 0: zero fill (rows beyond the chunk)
    if (sizeof(T) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
}

// B = 4 + BH row bits; rows 0 .. 2^B (the last one only for classes c < 2^B)
template <typename T, int BH>
__global__ void __launch_bounds__(SEAM_THREADS, 2) k_cvt_seam(CvtResParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    constexpr int W = sizeof(T) / 4;        // words per unit
    constexpr int C = 32 / W;               // classes per tile (one 128-byte row)
    constexpr int L = 16, H = 1 << BH, NB = 4 + BH, NR = (1 << NB) + 1;
    constexpr uint32_t BUF = (NR * 128 + 127) & ~127u;
    constexpr int I1 = (H + SEAM_NW - 1) / SEAM_NW;   // phase-1 items (row groups) per warp
    constexpr int I2 = L / SEAM_NW;                   // phase-2 items (low row index) per warp
    T* data = reinterpret_cast<T*>(p.data);
    const uint32_t M = (1u << p.K) - 1;
    const uint32_t span = 1u << p.q;
    const uint32_t nrb = (M + C - 1) / C;
    const uint64_t ntiles = (p.units_per_pair >> p.q) * p.batch * nrb;
    uint32_t* Qb = reinterpret_cast<uint32_t*>(smem_raw + 2 * BUF);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto prefetch = [&](uint64_t t, int b) {
        const uint64_t chunk = t / nrb;
        const uint32_t c0 = (uint32_t)(t - chunk * nrb) * C;
        const T* dp = data + (chunk << p.q);
        T* buf = reinterpret_cast<T*>(smem_raw + b * BUF);
        // SEAM_THREADS is a multiple of C: a thread keeps its class, its row advances by SEAM_THREADS / C
        const uint32_t c = c0 + 1 + threadIdx.x % C, di = (SEAM_THREADS / C) * M;
        uint32_t i = (threadIdx.x / C) * M + c;
        for (uint32_t s = threadIdx.x; s < (uint32_t)NR * C; s += SEAM_THREADS, i += di) {
            const bool ok = c <= M && i < span;
            seam_load_unit<T>(buf + s, dp + (ok ? i : 0), ok);
        }
    };
    if (blockIdx.x < ntiles) prefetch(blockIdx.x, 0);
    cp_async_commit();
    int kb = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, kb++) {
        if (t + gridDim.x < ntiles) prefetch(t + gridDim.x, (kb + 1) & 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        uint32_t* X = reinterpret_cast<uint32_t*>(smem_raw + (kb & 1) * BUF);
        const uint64_t chunk = t / nrb;
        const uint32_t c0 = (uint32_t)(t - chunk * nrb) * C;
        const uint32_t c = c0 + 1 + lane / W;   // this lane's class (> M: an empty column, never stored)
        if (!p.inverse) {
            // phase 1: row groups g (rows L g .. L g + L): low bits of P = S x (in place) and Q = T x (Qb)
            uint32_t v[I1][L + 1];
#pragma unroll
            for (int k = 0; k < I1; k++) {
                const int g = warp + k * SEAM_NW;
                if (g < H)
#pragma unroll
                    for (int u = 0; u <= L; u++) v[k][u] = X[(L * g + u) * 32 + lane];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < I1; k++) {
                const int g = warp + k * SEAM_NW;
                if (g < H) {
                    uint32_t q[L];
#pragma unroll
                    for (int u = 0; u < L; u++) q[u] = v[k][u + 1];
                    seam_ss<L>(v[k]);
                    seam_ss<L>(q);
#pragma unroll
                    for (int u = 0; u < L; u++) {
                        X[(L * g + u) * 32 + lane] = v[k][u];
                        Qb[(L * g + u) * 32 + lane] = q[u];
                    }
                }
            }
            __syncthreads();
            // phase 2: low index l (rows l + L h): high bits, the extra row 2^NB (a superset of row 0 only), the seam
            uint32_t pv[I2][H], qv[I2][H];
            const uint32_t xtra = X[(NR - 1) * 32 + lane];
#pragma unroll
            for (int k = 0; k < I2; k++) {
                const int l = warp + k * SEAM_NW;
#pragma unroll
                for (int h = 0; h < H; h++) {
                    pv[k][h] = X[(l + L * h) * 32 + lane];
                    qv[k][h] = Qb[(l + L * h) * 32 + lane];
                }
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < I2; k++) {
                const int l = warp + k * SEAM_NW;
                seam_ss<H>(pv[k]);
                seam_ss<H>(qv[k]);
                if (l == 0) pv[k][0] ^= xtra;
#pragma unroll
                for (int h = 0; h < H; h++) {
                    const uint32_t r = l + L * h;
                    if (r < c) X[r * 32 + lane] = pv[k][h];
                    if (r + 1 >= c) X[(r + 1) * 32 + lane] = qv[k][h];
                }
            }
        } else {
            // phase 1: low bits of T y (rows 1 .. 2^NB shifted down by one) -> Qb
            uint32_t v[I1][L];
#pragma unroll
            for (int k = 0; k < I1; k++) {
                const int g = warp + k * SEAM_NW;
                if (g < H) {
#pragma unroll
                    for (int u = 0; u < L; u++) v[k][u] = X[(L * g + u + 1) * 32 + lane];
                    seam_ss<L>(v[k]);
#pragma unroll
                    for (int u = 0; u < L; u++) Qb[(L * g + u) * 32 + lane] = v[k][u];
                }
            }
            __syncthreads();
            // phase 2: high bits of T y -> x_U (rows r = w + 1 >= c, into X); then the high bits of
            // S(x_U on U, 0 on L): the rows w + 1 of column l are column l + 1 (l = L - 1: column 0, one row group
            // up; its row 0 is in L, and the extra row 2^NB is only its own superset)
            uint32_t qv[I2][H];
#pragma unroll
            for (int k = 0; k < I2; k++) {
                const int l = warp + k * SEAM_NW;
#pragma unroll
                for (int h = 0; h < H; h++) qv[k][h] = Qb[(l + L * h) * 32 + lane];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < I2; k++) {
                const int l = warp + k * SEAM_NW;
                seam_ss<H>(qv[k]);
                uint32_t z[H];
                if (l < L - 1) {
#pragma unroll
                    for (int h = 0; h < H; h++) {
                        const uint32_t r = l + 1 + L * h;
                        const bool up = r >= c;
                        if (up) X[r * 32 + lane] = qv[k][h];
                        z[h] = up ? qv[k][h] : 0u;
                    }
                    seam_ss<H>(z);
#pragma unroll
                    for (int h = 0; h < H; h++) Qb[(l + 1 + L * h) * 32 + lane] = z[h];
                } else {
                    z[0] = 0u;
#pragma unroll
                    for (int h = 0; h < H; h++) {
                        const uint32_t r = L * (h + 1);
                        const bool up = r >= c;
                        if (up) X[r * 32 + lane] = qv[k][h];
                        if (h + 1 < H) z[h + 1] = up ? qv[k][h] : 0u;
                    }
                    const uint32_t zn = (uint32_t)(NR - 1) >= c ? qv[k][H - 1] : 0u;
                    seam_ss<H>(z);
#pragma unroll
                    for (int h = 0; h < H; h++) Qb[(L * h) * 32 + lane] = z[h];
                    Qb[(NR - 1) * 32 + lane] = zn;
                }
            }
            __syncthreads();
            // phase 3: low bits of S -> v; w = (y on L, v on U); low bits of S w -> Qb (own rows)
#pragma unroll
            for (int k = 0; k < I1; k++) {
                const int g = warp + k * SEAM_NW;
                if (g < H) {
                    uint32_t w[L];
#pragma unroll
                    for (int u = 0; u < L; u++) w[u] = Qb[(L * g + u) * 32 + lane];
                    seam_ss<L>(w);
#pragma unroll
                    for (int u = 0; u < L; u++) {
                        const uint32_t r = L * g + u;
                        if (r < c) w[u] = X[r * 32 + lane];
                    }
                    seam_ss<L>(w);
#pragma unroll
                    for (int u = 0; u < L; u++) Qb[(L * g + u) * 32 + lane] = w[u];
                }
            }
            __syncthreads();
            // phase 4: high bits of S w (+ the extra row v[2^NB] = x_U[2^NB] into row 0) -> x_L
            const uint32_t xtra = Qb[(NR - 1) * 32 + lane];
#pragma unroll
            for (int k = 0; k < I2; k++) {
                const int l = warp + k * SEAM_NW;
                uint32_t w[H];
#pragma unroll
                for (int h = 0; h < H; h++) w[h] = Qb[(l + L * h) * 32 + lane];
                seam_ss<H>(w);
                if (l == 0) w[0] ^= xtra;
#pragma unroll
                for (int h = 0; h < H; h++) {
                    const uint32_t r = l + L * h;
                    if (r < c) X[r * 32 + lane] = w[h];
                }
            }
        }
        __syncthreads();
        // store the tile's units
        {
            const T* buf = reinterpret_cast<const T*>(X);
            T* dp = data + (chunk << p.q);
            const uint32_t cc = c0 + 1 + threadIdx.x % C, di = (SEAM_THREADS / C) * M;
            if (cc <= M) {
                uint32_t i = (threadIdx.x / C) * M + cc;
                for (uint32_t s = threadIdx.x; s < (uint32_t)NR * C && i < span; s += SEAM_THREADS, i += di) dp[i] = buf[s];
            }
        }
        __syncthreads();   // the buffer is refilled by the prefetch two tiles on; Qb is rewritten next tile
    }
    cp_async_wait<0>();
}
static size_t seam_smem() { return 3 * (size_t)((257 * 128 + 127) & ~127); }

// ---------------------------------------------------------------------------------------------
// Register-blocked pass for a run of Taylor steps with K <= 4 (windows of <= 5 index bits) whose
// windows lie inside R <= 8 consecutive index bits [r_lo, r_lo + R) -- e.g. a whole CVT(8) node
// (12 steps).  XORs act on whole elements, so each 32-bit limb is independent: in a phase a thread
// holds one limb of the 2^WB elements spanned by WB consecutive row bits [w_lo, w_lo + WB) and runs
// every step of that phase in registers (straight-line code per (K, window offset)); phases
// exchange data through the shared-memory tile.  A CVT(8) takes 3 phases instead of 12 steps x 2
// shared-memory sweeps.
//   mode 0: tile = columns (index bits [0, C), contiguous) x rows (bits [r_lo, r_lo + R)), r_lo >= C
//   mode 1: tile = rows (bits [0, R)) x columns (bits [R, R + C)); shared rows padded by one element
// ---------------------------------------------------------------------------------------------
#define RB_MAX_PHASES 6
#define RB_PAD(T) (16 / (uint32_t)sizeof(T))   // mode-1 column padding (16 B keeps bulk copies aligned)
#define RB_MAX_OPS 48
struct CvtRbParams {
    void* data;
    uint64_t units_per_pair, batch;
    int r_lo, R, C, mode, inverse;
    int nphase;
    int st_tma;                  // k_cvt_rb_tma: 0 = thread stores; 1 = TMA stores, next load issued at the
                                 // iteration start; 2 = TMA stores, next load issued after the first phase
    int ph_lo[RB_MAX_PHASES];    // phase window [ph_lo, ph_lo + WB) in row-bit coordinates
    int ph_n[RB_MAX_PHASES];     // ops per phase
    unsigned char ops[RB_MAX_OPS];   // (K index: 0 -> K=1, 1 -> K=2, 2 -> K=4) | (offset in the phase window << 2)
};

// one Taylor step with window bits [OFF, OFF + K + 1) of the WB-bit register block
template <int WB, int K, int OFF, bool INV>
__device__ __forceinline__ void rb_step(uint32_t* v) {
    constexpr int T = 1 << K;
#pragma unroll
    for (int rest = 0; rest < (1 << WB); rest++) {
        if ((rest >> OFF) & ((2 << K) - 1)) continue;   // enumerate the other bits only
        auto at = [&](int y) -> uint32_t& { return v[rest | (y << OFF)]; };
        if (!INV) {
            at(T) ^= at(2 * T - 1);
#pragma unroll
            for (int y = 1; y < T; y++) at(y) ^= at(y + T - 1);
        } else {
#pragma unroll
            for (int y = 1; y < T; y++) at(y) ^= at(y + T - 1);
            at(T) ^= at(2 * T - 1);
        }
    }
}

template <int WB, bool INV>
__device__ __forceinline__ void rb_dispatch(uint32_t* v, int code) {
    const int kk = code & 3, off = code >> 2;
    // K = 1 (2-bit windows)
    if (kk == 0) {
        if (off == 0) { if (WB >= 2) rb_step<WB, 1, 0, INV>(v); }
        else if (off == 1) { if (WB >= 3) rb_step<WB, 1, (WB >= 3 ? 1 : 0), INV>(v); }
        else if (off == 2) { if (WB >= 4) rb_step<WB, 1, (WB >= 4 ? 2 : 0), INV>(v); }
        else if (off == 3) { if (WB >= 5) rb_step<WB, 1, (WB >= 5 ? 3 : 0), INV>(v); }
        else { if (WB >= 6) rb_step<WB, 1, (WB >= 6 ? 4 : 0), INV>(v); }
    } else if (kk == 1) {   // K = 2 (3-bit windows)
        if (off == 0) { if (WB >= 3) rb_step<WB, (WB >= 3 ? 2 : 1), 0, INV>(v); }
        else if (off == 1) { if (WB >= 4) rb_step<WB, (WB >= 4 ? 2 : 1), (WB >= 4 ? 1 : 0), INV>(v); }
        else if (off == 2) { if (WB >= 5) rb_step<WB, (WB >= 5 ? 2 : 1), (WB >= 5 ? 2 : 0), INV>(v); }
        else { if (WB >= 6) rb_step<WB, (WB >= 6 ? 2 : 1), (WB >= 6 ? 3 : 0), INV>(v); }
    } else {                // K = 4 (5-bit windows)
        if (off == 0) { if (WB >= 5) rb_step<WB, (WB >= 5 ? 4 : 1), 0, INV>(v); }
        else { if (WB >= 6) rb_step<WB, (WB >= 6 ? 4 : 1), (WB >= 6 ? 1 : 0), INV>(v); }
    }
}

template <typename T, int WB>
__device__ __forceinline__ void rb_phase(uint32_t* s32, const CvtRbParams& p, int ph, int op0) {
    constexpr int LW = sizeof(T) / 4;   // 32-bit limbs per unit
    const int w_lo = p.ph_lo[ph];
    const int nrest = p.R - WB;         // row bits outside the phase window
    const uint32_t items = (uint32_t)LW << (p.C + nrest);
    const uint32_t rowstride = p.mode ? 1u : (1u << p.C);
    const uint32_t colstride = p.mode ? ((1u << p.R) + RB_PAD(T)) : 1u;
    for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
        const uint32_t L = it % LW, rest = it / LW;
        const uint32_t col = rest & ((1u << p.C) - 1), rr = rest >> p.C;
        // row bits outside [w_lo, w_lo + WB): low part below w_lo, high part above
        const uint32_t rfix = (rr & ((1u << w_lo) - 1)) | ((rr >> w_lo) << (w_lo + WB));
        const uint32_t base = (rfix * rowstride + col * colstride) * LW + L;
        const uint32_t jstride = (rowstride << w_lo) * LW;
        uint32_t v[1 << WB];
#pragma unroll
        for (int j = 0; j < (1 << WB); j++) v[j] = s32[base + j * jstride];
        for (int o = 0; o < p.ph_n[ph]; o++) {
            const int code = p.ops[op0 + ((p.inverse & 1) ? p.ph_n[ph] - 1 - o : o)];
            if (p.inverse & 1) rb_dispatch<WB, true>(v, code);
            else rb_dispatch<WB, false>(v, code);
        }
#pragma unroll
        for (int j = 0; j < (1 << WB); j++) s32[base + j * jstride] = v[j];
    }
}

#define RB_THREADS 128
// Double-buffered: the next tile is prefetched with cp.async (16-byte pieces of the tile's contiguous
// runs, straight into shared memory) while the current one runs its phases; tiles are stored from
// shared memory with ordinary vector stores.  (A variant with cp.async.bulk row copies issued by one
// warp measured 3x slower on B200: 256-byte bulk copies are issue-bound.)  p.inverse bit 1
// (GF2X_RB_NOPHASE, measurement only) skips the phases.
template <typename T>
__device__ __forceinline__ void rb_slot(const CvtRbParams& p, uint32_t s, uint64_t base, uint32_t& sm, uint64_t& g) {
    const uint32_t nrows = 1u << p.R, ncols = 1u << p.C;
    if (p.mode) { const uint32_t row = s & (nrows - 1), col = s >> p.R; sm = col * (nrows + RB_PAD(T)) + row; g = base + s; }
    else { const uint32_t col = s & (ncols - 1), row = s >> p.C; sm = s; g = base + col + ((uint64_t)row << p.r_lo); }
}

template <typename T, int WB>
__device__ __forceinline__ void cvt_rb_tiles(const CvtRbParams& p, T* data, uint64_t t_first, uint64_t t_step,
                                             unsigned char* smem_raw) {
    constexpr uint32_t EPC = 16 / sizeof(T);   // units per 16-byte copy
    const uint32_t ncols = 1u << p.C, nrows = 1u << p.R, nslots = ncols << p.R;
    const uint32_t bufsz = ((ncols * (nrows + (p.mode ? RB_PAD(T) : 0)) * (uint32_t)sizeof(T)) + 127) & ~127u;
    // (buffers are addressed from smem_raw directly so the compiler emits LDS/STS, not generic LD/ST)
    const uint64_t tiles_per_pair = p.units_per_pair >> (p.R + p.C);
    const uint64_t ntiles = tiles_per_pair * p.batch;
    const int midbits = p.mode ? 0 : p.r_lo - p.C;
    auto tile_at = [&](uint64_t t, T*& dp, uint64_t& base) {
        const uint64_t pair = t / tiles_per_pair, tt = t - pair * tiles_per_pair;
        dp = data + pair * p.units_per_pair;
        if (p.mode) base = tt << (p.R + p.C);
        else base = ((tt & ((1ull << midbits) - 1)) << p.C) | ((tt >> midbits) << (p.r_lo + p.R));
    };
    // a thread's slots s = tid EPC + k S (S = threads EPC, a multiple of the tile's column count) advance the
    // global pointer by a constant stride: strength-reduced 64-bit addressing in the copy loops
    const uint32_t S = blockDim.x * EPC;
    const uint64_t gstride = p.mode ? (uint64_t)S : ((uint64_t)(S >> p.C) << p.r_lo);
    auto prefetch = [&](uint64_t t, T* buf) {
        T* dp; uint64_t base;
        tile_at(t, dp, base);
        uint32_t s = threadIdx.x * EPC, sm;
        uint64_t g;
        rb_slot<T>(p, s, base, sm, g);
        const T* gp = dp + g;
        for (; s < nslots; s += S, gp += gstride) {
            rb_slot<T>(p, s, 0, sm, g);
            cp_async16(buf + sm, gp);
        }
    };
    if (t_first < ntiles) prefetch(t_first, reinterpret_cast<T*>(smem_raw));
    cp_async_commit();
    int k = 0;
    for (uint64_t t = t_first; t < ntiles; t += t_step, k++) {
        T* buf = reinterpret_cast<T*>(smem_raw + (k & 1) * bufsz);
        if (t + t_step < ntiles) prefetch(t + t_step, reinterpret_cast<T*>(smem_raw + ((k + 1) & 1) * bufsz));
        cp_async_commit();
        cp_async_wait<1>();   // this tile's copies (all but the newest group) have landed
        __syncthreads();
        uint32_t* s32 = reinterpret_cast<uint32_t*>(smem_raw + (k & 1) * bufsz);
        for (int i = 0; i < p.nphase * (p.inverse >> 1 ? 0 : 1); i++) {
            const int ph = (p.inverse & 1) ? p.nphase - 1 - i : i;
            int o0 = 0;
            for (int q = 0; q < ph; q++) o0 += p.ph_n[q];
            rb_phase<T, WB>(s32, p, ph, o0);
            __syncthreads();
        }
        T* dp; uint64_t base;
        tile_at(t, dp, base);
        {
            uint32_t s = threadIdx.x * EPC, sm;
            uint64_t g;
            rb_slot<T>(p, s, base, sm, g);
            T* gp = dp + g;
            for (; s < nslots; s += S, gp += gstride) {
                rb_slot<T>(p, s, 0, sm, g);
                *reinterpret_cast<uint4*>(gp) = *reinterpret_cast<const uint4*>(buf + sm);
            }
        }
        __syncthreads();   // the buffer is refilled by the prefetch two tiles on
    }
    cp_async_wait<0>();
}

template <typename T, int WB>
__global__ void __launch_bounds__(RB_THREADS, 3) k_cvt_rb(CvtRbParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    cvt_rb_tiles<T, WB>(p, reinterpret_cast<T*>(p.data), blockIdx.x, gridDim.x, smem_raw);
}

// The same pass with the tile loads done by the TMA engine (SURVEY §8a "TMA bulk copies into smem"): one
// thread per CTA issues, per tile, one 4-D tensor-map load (mode 0: 2^C contiguous units x 2^R rows at stride
// 2^r_lo units; dims (units of the column run, middle bits, rows, rest)) or one 1-D bulk copy per column
// (mode 1: the tile is 2^C contiguous runs of 2^R units, each landing after its column's shared-memory pad);
// the copies complete on the buffer's mbarrier (transaction count = tile bytes).  Replaces 2^(R+C)/EPC
// cp.async instructions and their address arithmetic per tile.  Stores (p.st_tma, default 2): the same tensor
// map / 2^C bulk copies in the other direction, issued by thread 0 after the last phase; the next tile's load
// into the other buffer waits (cp.async.bulk.wait_group.read) for the previous store to have read it, issued
// after the first phase (c4b: 0.074 -> 0.068 ms per pass against thread stores; 1 = issued at the iteration
// start: 0.071).
template <typename T, int WB>
__global__ void __launch_bounds__(RB_THREADS, 3) k_cvt_rb_tma(CvtRbParams p, const __grid_constant__ CUtensorMap tm) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];
    T* data = reinterpret_cast<T*>(p.data);
    constexpr uint32_t EPC = 16 / sizeof(T);
    const uint32_t ncols = 1u << p.C, nrows = 1u << p.R, nslots = ncols << p.R;
    const uint32_t bufsz = ((ncols * (nrows + (p.mode ? RB_PAD(T) : 0)) * (uint32_t)sizeof(T)) + 127) & ~127u;
    const uint64_t tiles_per_pair = p.units_per_pair >> (p.R + p.C);
    const uint64_t ntiles = tiles_per_pair * p.batch;
    const int midbits = p.mode ? 0 : p.r_lo - p.C;
    const uint64_t rest_per_pair = p.units_per_pair >> (p.r_lo + p.R);
    auto tile_at = [&](uint64_t t, T*& dp, uint64_t& base) {
        const uint64_t pair = t / tiles_per_pair, tt = t - pair * tiles_per_pair;
        dp = data + pair * p.units_per_pair;
        if (p.mode) base = tt << (p.R + p.C);
        else base = ((tt & ((1ull << midbits) - 1)) << p.C) | ((tt >> midbits) << (p.r_lo + p.R));
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto prefetch = [&](uint64_t t, int b) {   // thread 0 only
        T* buf = reinterpret_cast<T*>(smem_raw + b * bufsz);
        fence_proxy_async_smem();   // the buffer's earlier generic-proxy reads / writes come first
        mbar_arrive_expect_tx(&bars[b], nslots * (uint32_t)sizeof(T));
        const uint64_t pair = t / tiles_per_pair, tt = t - pair * tiles_per_pair;
        if (p.mode) {
            const T* src = data + pair * p.units_per_pair + (tt << (p.R + p.C));
            for (uint32_t col = 0; col < ncols; col++)
                bulk_g2s(buf + col * (nrows + RB_PAD(T)), src + ((uint64_t)col << p.R), nrows * (uint32_t)sizeof(T), &bars[b]);
        } else {
            tma_load_4d(buf, &tm, 0, (int)(tt & ((1ull << midbits) - 1)), 0,
                        (int)(pair * rest_per_pair + (tt >> midbits)), &bars[b]);
        }
    };
    // TMA stores (p.st_tma): the tile leaves shared memory by one tensor store (mode 0) or 2^C bulk stores
    // (mode 1) issued by thread 0 after the last phase; a buffer is refilled only after the bulk stores that
    // read it have read it (cp.async.bulk.wait_group.read), so the store drains while the next tile's phases run
    auto store_tile = [&](uint64_t t, int b) {   // thread 0 only
        const T* buf = reinterpret_cast<const T*>(smem_raw + b * bufsz);
        const uint64_t pair = t / tiles_per_pair, tt = t - pair * tiles_per_pair;
        if (p.mode) {
            T* dst = data + pair * p.units_per_pair + (tt << (p.R + p.C));
            for (uint32_t col = 0; col < ncols; col++)
                bulk_s2g(dst + ((uint64_t)col << p.R), buf + col * (nrows + RB_PAD(T)), nrows * (uint32_t)sizeof(T));
        } else {
            tma_store_4d(&tm, 0, (int)(tt & ((1ull << midbits) - 1)), 0, (int)(pair * rest_per_pair + (tt >> midbits)), buf);
        }
        bulk_commit();
    };
    const int stm = p.st_tma;
    if (threadIdx.x == 0 && blockIdx.x < ntiles) prefetch(blockIdx.x, 0);
    const uint32_t S = blockDim.x * EPC;
    const uint64_t gstride = p.mode ? (uint64_t)S : ((uint64_t)(S >> p.C) << p.r_lo);
    int k = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, k++) {
        const int b = k & 1;
        T* buf = reinterpret_cast<T*>(smem_raw + b * bufsz);
        const bool has_next = t + gridDim.x < ntiles;
        if (threadIdx.x == 0 && has_next && (stm != 2 || p.nphase == 0)) {
            if (stm) bulk_wait_read<0>();   // the previous tile's store has read buffer b ^ 1
            prefetch(t + gridDim.x, b ^ 1);
        }
        mbar_wait(&bars[b], (uint32_t)(k >> 1) & 1);   // this tile has landed
        uint32_t* s32 = reinterpret_cast<uint32_t*>(smem_raw + b * bufsz);
        for (int i = 0; i < p.nphase; i++) {
            const int ph = (p.inverse & 1) ? p.nphase - 1 - i : i;
            int o0 = 0;
            for (int q = 0; q < ph; q++) o0 += p.ph_n[q];
            rb_phase<T, WB>(s32, p, ph, o0);
            if (stm) fence_proxy_async_smem();   // the phase's writes before the TMA store's reads
            __syncthreads();
            if (i == 0 && stm == 2 && threadIdx.x == 0 && has_next) {
                bulk_wait_read<0>();
                prefetch(t + gridDim.x, b ^ 1);
            }
        }
        if (stm) {
            if (threadIdx.x == 0) store_tile(t, b);
            continue;   // the buffer is refilled after the store has read it (wait above)
        }
        T* dp; uint64_t base;
        tile_at(t, dp, base);
        {
            uint32_t s = threadIdx.x * EPC, sm;
            uint64_t g;
            rb_slot<T>(p, s, base, sm, g);
            T* gp = dp + g;
            for (; s < nslots; s += S, gp += gstride) {
                rb_slot<T>(p, s, 0, sm, g);
                *reinterpret_cast<uint4*>(gp) = *reinterpret_cast<const uint4*>(buf + sm);
            }
        }
        __syncthreads();   // the buffer is refilled by the prefetch two tiles on
    }
    if (stm && threadIdx.x == 0) bulk_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// Top Taylor run of a conversion (k_cvt_top): the whole Taylor part of CVT(q) with K = 16 (levels
// q .. K+1 of a 2^q-unit chunk; Alg. 3 l.531 with Alg. 2's divisions), as residue classes
// i = r M + c (M = 2^K - 1, R17) in tiles of 2^C_log classes x all rows.
//
// With B = q - K row bits, write i = r 2^K + (c - r) for r <= c.  Level l (u = 2^(l-1-K), h = u 2^K) makes
// the units at position (i mod 2^l) in [u, h + u) targets of f[t] ^= f[t + u M] -- the source is row r + u
// of the same class.  For every class c >= 2^B - 1 + 2^(B-1) ("generic"; all but the first ~1.5 2^B of the
// 2^K - 1 classes) the class has exactly 2^B rows, all r <= c with c - r >= u, and the position test reduces
// to (r mod 2u) < u, i.e. bit log2(u) of r is clear.  The run on such a class is therefore
//     for every row bit b (any order):  x[r] ^= x[r + 2^b]  for r with bit b clear,
// the superset-sum transform over the B row bits: data-independent, its steps commute, and it is its own
// inverse (the inverse run is the same transform).  Generic tiles run it register-blocked, <= 4 row bits per
// phase through shared memory.  Tiles holding the first classes run Alg. 2's steps exactly, one sweep per
// phase (A: targets [h, h+u), B: [u, h); forward A then B, inverse B then A, levels in Alg. 3's order), as
// k_cvt_res does.  Pinned by the stage / end-to-end parity tests against the oracle's Alg. 3.
//
// Split can be fused into a forward run: the tile is then read from the caller's operand
// words (pairs [0, batch0) from src0, the rest from src1; words >= nsrc read as 0, the last one masked
// to `bits`) instead of the scratch array it writes.
// ---------------------------------------------------------------------------------------------
struct CvtTopParams {
    void* data;
    uint64_t units_per_pair, batch;   // one chunk per pair: units_per_pair = 2^q
    int q, K, B, inverse, C_log;
    uint32_t c_gen;                   // classes >= c_gen take the transform path
    const uint64_t* src0;             // fused Split (T = u64, forward): operand words, or null
    const uint64_t* src1;
    uint64_t batch0, nsrc, bits;
};
#define TOP_THREADS 256

template <int NB>
__device__ __forceinline__ void top_phase(uint32_t* s32, uint32_t items, int b0, int Bt, uint32_t WC) {
    // item = (word w of the unit, class c) fastest (contiguous words across lanes), then the row bits
    // outside [b0, b0 + NB); the NB row bits in [b0, b0 + NB) are the register dimension
    const uint32_t rowstride = WC;   // words per tile row
    for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
        const uint32_t wc = it % WC, rest = it / WC;
        const uint32_t r0 = (rest & ((1u << b0) - 1)) | ((rest >> b0) << (b0 + NB));
        uint32_t* p = s32 + r0 * rowstride + wc;
        const uint32_t js = (rowstride << b0);
        uint32_t v[1 << NB];
#pragma unroll
        for (int j = 0; j < (1 << NB); j++) v[j] = p[j * js];
#pragma unroll
        for (int k = 0; k < NB; k++)
#pragma unroll
            for (int j = 0; j < (1 << NB); j++)
                if (!(j & (1 << k))) v[j] ^= v[j | (1 << k)];
#pragma unroll
        for (int j = 0; j < (1 << NB); j++) p[j * js] = v[j];
    }
    (void)Bt;
}

template <typename T>
__global__ void __launch_bounds__(TOP_THREADS, 2) k_cvt_top(CvtTopParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    T* data = reinterpret_cast<T*>(p.data);
    constexpr uint32_t W = sizeof(T) / 4;   // 32-bit words per unit
    const uint32_t M = (1u << p.K) - 1;
    const uint32_t C = 1u << p.C_log;
    const uint32_t nrb = (M + C - 1) >> p.C_log;
    const uint32_t rows = (1u << p.B) + 1;
    const uint32_t span = 1u << p.q;
    const uint64_t ntiles = p.batch * nrb;
    const uint32_t nslots = rows << p.C_log;
    const uint32_t bufsz = (nslots * (uint32_t)sizeof(T) + 127) & ~127u;
    const bool fuse = p.src0 != nullptr;   // (T = u64)
    const uint32_t rem = (uint32_t)(p.bits & 63);
    auto prefetch = [&](uint64_t t, T* buf) {
        const uint64_t pair = t / nrb;
        const uint32_t c0 = (uint32_t)(t - pair * nrb) << p.C_log;
        T* dp = data + pair * p.units_per_pair;
        const uint64_t* sp = fuse ? (pair < p.batch0 ? p.src0 + pair * p.nsrc : p.src1 + (pair - p.batch0) * p.nsrc) : nullptr;
        // blockDim is a multiple of C: a thread keeps its class, its row advances by blockDim / C (units i by that
        // times M; rows only grow, so the first one past the chunk ends the loop)
        const uint32_t c = c0 + (threadIdx.x & (C - 1));
        if (c >= M) return;
        const uint32_t di = (blockDim.x >> p.C_log) * M;
        uint32_t i = (threadIdx.x >> p.C_log) * M + c;
        for (uint32_t s = threadIdx.x; s < nslots && i < span; s += blockDim.x, i += di) {
            if (fuse) {
                const uint32_t n = (uint64_t)i < p.nsrc ? 8u : 0u;   // src-size 0: zero fill (words >= nsrc)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(buf + s)),
                             "l"(sp + (i < p.nsrc ? i : 0)), "r"(n) : "memory");
            } else {
                cp_async_unit<T>(buf + s, dp + i);
            }
        }
    };
    if (blockIdx.x < ntiles) prefetch(blockIdx.x, reinterpret_cast<T*>(smem_raw));
    cp_async_commit();
    int kb = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, kb++) {
        if (t + gridDim.x < ntiles) prefetch(t + gridDim.x, reinterpret_cast<T*>(smem_raw + ((kb + 1) & 1) * bufsz));
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        T* tile = reinterpret_cast<T*>(smem_raw + (kb & 1) * bufsz);
        const uint64_t pair = t / nrb;
        const uint32_t c0 = (uint32_t)(t - pair * nrb) << p.C_log;
        if (fuse && rem && p.nsrc && (uint32_t)((p.nsrc - 1) % M) - c0 < C) {
            // the operand's last word lies in this tile: clear its bits >= bits (Split's mask)
            if (threadIdx.x == 0) {
                const uint32_t i = (uint32_t)(p.nsrc - 1);
                uint64_t* w = reinterpret_cast<uint64_t*>(tile) + (((i / M) << p.C_log) | (i % M - c0));
                *w &= (1ull << rem) - 1;
            }
            __syncthreads();
        }
        if (c0 >= p.c_gen) {
            // superset-sum transform over the B row bits, <= 4 bits per phase
            uint32_t* s32 = reinterpret_cast<uint32_t*>(tile);
            const uint32_t WC = W << p.C_log;
            for (int b0 = 0; b0 < p.B; b0 += 4) {
                const int nb = min(4, p.B - b0);
                const uint32_t items = WC << (p.B - nb);
                if (nb == 4) top_phase<4>(s32, items, b0, p.B, WC);
                else if (nb == 3) top_phase<3>(s32, items, b0, p.B, WC);
                else if (nb == 2) top_phase<2>(s32, items, b0, p.B, WC);
                else top_phase<1>(s32, items, b0, p.B, WC);
                __syncthreads();
            }
        } else {
            // Alg. 2's steps exactly: per level the phase-A sweep (targets [h, h+u)) and the phase-B sweep
            // ([u, h)), each f[t] ^= f[t + u M] = row r + u of the class
            const int nl = p.q - p.K;
            for (int o = 0; o < nl; o++) {
                const int lg = p.inverse ? p.K + 1 + o : p.q - o;
                const uint32_t u = 1u << (lg - 1 - p.K), h = 1u << (lg - 1), segm = (lg >= 32) ? 0xFFFFFFFFu : ((1u << lg) - 1);
                for (int ph = 0; ph < 2; ph++) {
                    const bool A = (ph == 0) != (p.inverse != 0);
                    const uint32_t lo = A ? h : u, len = A ? u : h - u;
                    for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x) {
                        const uint32_t r = s >> p.C_log, c = c0 + (s & (C - 1));
                        const uint32_t i = r * M + c;
                        if (c >= M || i >= span) continue;
                        if (((i & segm) - lo) < len) tile[s] = xor_t<T>(tile[s], tile[s + (u << p.C_log)]);
                    }
                    __syncthreads();
                }
            }
        }
        T* dp = data + pair * p.units_per_pair;
        {
            const uint32_t c = c0 + (threadIdx.x & (C - 1));
            if (c < M) {
                const uint32_t di = (blockDim.x >> p.C_log) * M;
                uint32_t i = (threadIdx.x >> p.C_log) * M + c;
                for (uint32_t s = threadIdx.x; s < nslots && i < span; s += blockDim.x, i += di) dp[i] = tile[s];
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// CVT(16) slab pass (k_cvt_slab): the inner conversion of the top node on every 2^16-unit slab -- its
// K = 8 Taylor run (levels 16 .. 9, residue classes mod 255, R17) and its two CVT(8) nodes (bits [0, 8) and
// [8, 16), register-blocked, R18) -- in ONE launch instead of three HBM passes (SURVEY §8(d) P3's slab).
// A thread-block cluster owns one slab at a time: each phase's tiles are split over the cluster's CTAs, and
// the phases are separated by cluster barriers (barrier.cluster arrive.release / wait.acquire: the global
// writes of one phase are visible to every CTA of the cluster in the next one; the acquire invalidates L1).
// The slab (512 KB u64 / 1 MB u128) stays in L2 between the phases, so HBM sees one read and one write per
// unit; the ~18 slabs in flight are far below the 126 MB L2.  Same device code as k_cvt_res / k_cvt_rb.
// Order (Alg. 3, with R14): forward Taylor run, CVT(8) [0,8), CVT(8) [8,16); inverse reversed.
// ---------------------------------------------------------------------------------------------
struct CvtSlabParams {
    void* data;
    uint64_t nslabs;
    CvtResParams res;     // data / units_per_pair / batch set per slab
    CvtRbParams rb_lo;    // CVT(8) on bits [0, 8)
    CvtRbParams rb_hi;    // CVT(8) on bits [8, 16)
    int inverse;
};
#define SLAB_THREADS 256
#define SLAB_BITS 16
#ifndef SLAB_MINB
#define SLAB_MINB 2
#endif

template <typename T>
__global__ void __launch_bounds__(SLAB_THREADS, SLAB_MINB) k_cvt_slab(CvtSlabParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint32_t cs, cr;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
    const uint64_t ncl = gridDim.x / cs, cid = blockIdx.x / cs;
    T* data = reinterpret_cast<T*>(P.data);
    auto csync = [] {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    };
    for (uint64_t sl = cid; sl < P.nslabs; sl += ncl) {
        T* base = data + (sl << SLAB_BITS);
        if (!P.inverse) {
            cvt_res_tiles<T>(P.res, base, cr, cs, smem_raw);
            csync();
            cvt_rb_tiles<T, 6>(P.rb_lo, base, cr, cs, smem_raw);
            csync();
            cvt_rb_tiles<T, 6>(P.rb_hi, base, cr, cs, smem_raw);
        } else {
            cvt_rb_tiles<T, 6>(P.rb_hi, base, cr, cs, smem_raw);
            csync();
            cvt_rb_tiles<T, 6>(P.rb_lo, base, cr, cs, smem_raw);
            csync();
            cvt_res_tiles<T>(P.res, base, cr, cs, smem_raw);
        }
        csync();   // (the next slab's first phase reuses shared memory only after every CTA left this one)
    }
}
