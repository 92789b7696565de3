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

template <typename T>
__global__ void __launch_bounds__(512) k_cvt_res(CvtResParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw);
    T* data = reinterpret_cast<T*>(p.data);
    const uint32_t M = (1u << p.K) - 1;
    const uint32_t C = 1u << p.C_log, cmask = C - 1;
    const uint32_t nrb = (M + C - 1) >> p.C_log;
    const uint32_t span = 1u << p.q;                       // q <= 31
    const uint64_t chunks = (p.units_per_pair >> p.q) * p.batch;
    const uint64_t ntiles = chunks * nrb;
    const uint32_t nslots = (uint32_t)p.rows << p.C_log;
    const int nsteps = p.lg_hi - p.lg_lo + 1;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t chunk = t / nrb;
        const uint32_t c0 = (uint32_t)(t - chunk * nrb) << p.C_log;
        const uint32_t cn = min(C, M - c0);
        T* dp = data + chunk * span;
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x) {
            const uint32_t c = s & cmask, i = (s >> p.C_log) * M + c0 + c;
            if (c < cn && i < span) tile[s] = dp[i];
        }
        __syncthreads();
        for (int o = 0; o < nsteps; o++) {
            const int lg = p.inverse ? p.lg_lo + o : p.lg_hi - o;
            const uint32_t h = 1u << (lg - 1), u = h >> p.K, segm = (2u << (lg - 1)) - 1;
            const uint32_t off = u << p.C_log;
            for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x) {
                const uint32_t c = s & cmask, i = (s >> p.C_log) * M + c0 + c;
                const uint32_t pos = i & segm;
                if (c >= cn || i >= span || pos < u || pos >= h) continue;
                if (pos < 2 * u) {   // also owns the phase-A target s + off
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
            __syncthreads();
        }
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x) {
            const uint32_t c = s & cmask, i = (s >> p.C_log) * M + c0 + c;
            if (c < cn && i < span) dp[i] = tile[s];
        }
        __syncthreads();
    }
}
