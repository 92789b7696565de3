// bottom.cuh -- fused bottom kernel, included by gf2x.cu: the FFT_LCH layers L-1..0 of both spectra
// (Alg. 1), pointmul and the iFFT_LCH layers 0..L-1, L = min(m, 6),
// on tiles of 2^11 consecutive elements, entirely in bit-sliced form (SURVEY §8d pass P3).
//
// Layout of a tile (flattened element index g over all pairs, bits [0,11) of it):
//   bits [0, L)        -> "word" bits: the butterfly dimensions of the bottom layers
//   bits [L, L+5)      -> bit position inside a 32-bit plane word (32 elements per group)
//   bits [L+5, 11)     -> more groups
// A group = 32 elements sharing bits outside [L, L+5); its limb Lb is held as 32 planes (plane j =
// bit j of the 32 limbs).  Butterflies at layer k < L pair groups g and g ^ 2^k at the same bit
// positions, so a butterfly of 32 elements is one bit-sliced multiply by the 32 per-position
// multipliers s_k(phi(b)).  By linearity (s_k is GF(2)-linear, A10) the multiplier planes are
//   c_j = P_k[j] ^ (bit j of U_k(g) ? ~0 : 0),
// P_k[j] = XOR over position bits i of (bit j of s_k(v_(L+i))) * POS_i   (fixed per layer),
// U_k(g) = s_k(phi(the group's bits above k outside the position bits))  (one scalar per group).
// Planes of block (group g, limb Lb) live at word ((Lb * 64 + g) * 33 + j).
#pragma once

#define BT_THREADS 128
#define BT_BITS 11
#define BT_GROUPS 64
#define BT_STRIDE 33
#define BT_REGION (4 * BT_GROUPS * BT_STRIDE)   // words per operand region

struct BottomParams {
    uint4* A;            // spectrum of a (in: after the direct passes; out: product, after iFFT bottom)
    uint4* B;            // spectrum of b
    uint64_t total;      // batch * N elements per operand (A and B may be adjacent: never touch beyond)
    uint64_t ntiles;     // ceil(total / 2^11)
    int m, L, mode;      // mode bit0: forward layers, bit1: pointmul, bit2: inverse layers
};

__device__ __forceinline__ uint32_t bt_block(int g, int lb) { return (uint32_t)((lb * BT_GROUPS + g) * BT_STRIDE); }

// element (within the tile) of group g at bit position p
__device__ __forceinline__ uint32_t bt_elem(int g, int p, int L) {
    return (uint32_t)((g & ((1 << L) - 1)) | (p << L) | ((g >> L) << (L + 5)));
}

// global -> planes of (group g, limb lb)
__device__ __forceinline__ void bt_load_block(const uint4* __restrict__ src, uint64_t e0, uint64_t total, int g, int lb,
                                              int L, uint32_t* planes) {
    uint32_t x[32];
    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
#pragma unroll
    for (int p = 0; p < 32; p++) {
        const uint64_t e = e0 + bt_elem(g, p, L);
        x[p] = e < total ? s32[e * 4 + lb] : 0u;
    }
    transpose32(x);
    uint32_t* d = planes + bt_block(g, lb);
#pragma unroll
    for (int j = 0; j < 32; j++) d[j] = x[j];
}

__device__ __forceinline__ void bt_store_block(uint4* __restrict__ dst, uint64_t e0, uint64_t total, int g, int lb, int L,
                                               const uint32_t* planes) {
    uint32_t x[32];
    const uint32_t* s = planes + bt_block(g, lb);
#pragma unroll
    for (int j = 0; j < 32; j++) x[j] = s[j];
    transpose32(x);
    uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
#pragma unroll
    for (int p = 0; p < 32; p++) {
        const uint64_t e = e0 + bt_elem(g, p, L);
        if (e < total) d32[e * 4 + lb] = x[p];
    }
}

// one layer k of butterflies on a plane region: warp = limb, lane = pair index
template <bool INV>
__device__ __forceinline__ void bt_layer(uint32_t* planes, int k, const uint32_t* Pk, uint64_t e0, int L, int m) {
    const int lb = threadIdx.x >> 5, q = threadIdx.x & 31;
    const int g0 = (q & ((1 << k) - 1)) | ((q >> k) << (k + 1));
    const int g1 = g0 | (1 << k);
    // U_k(g0): within-pair index of the group's block base with the position bits cleared
    const uint64_t N = 1ull << m;
    const uint64_t gi = (e0 + bt_elem(g0, 0, L)) & (N - 1);
    const uint32_t U = layer_const(k, (uint32_t)gi);
    uint32_t c[32], x1[32], pr[32];
#pragma unroll
    for (int j = 0; j < 32; j++) c[j] = Pk[j] ^ (((U >> j) & 1) ? 0xFFFFFFFFu : 0u);
    uint32_t* b0 = planes + bt_block(g0, lb);
    uint32_t* b1 = planes + bt_block(g1, lb);
#pragma unroll
    for (int j = 0; j < 32; j++) x1[j] = b1[j];
    if (INV) {
#pragma unroll
        for (int j = 0; j < 32; j++) x1[j] ^= b0[j];
    }
    bs_mul32(x1, c, pr);
#pragma unroll
    for (int j = 0; j < 32; j++) {
        const uint32_t x0 = b0[j] ^ pr[j];
        b0[j] = x0;
        b1[j] = INV ? x1[j] : (x1[j] ^ x0);
    }
}

// pointmul on one group (see k_pointmul for the limb formulas); planes of limb L of group g
__device__ __forceinline__ void bt_load_sum(const uint32_t* reg, int g, int mask, uint32_t* x) {
#pragma unroll
    for (int j = 0; j < 32; j++) x[j] = 0;
#pragma unroll
    for (int l = 0; l < 4; l++)
        if (mask & (1 << l)) {
            const uint32_t* s = reg + bt_block(g, l);
#pragma unroll
            for (int j = 0; j < 32; j++) x[j] ^= s[j];
        }
}
__device__ __forceinline__ void bt_acc_add(uint32_t* reg, int g, int mask, const uint32_t* v) {
#pragma unroll
    for (int l = 0; l < 4; l++)
        if (mask & (1 << l)) {
            uint32_t* d = reg + bt_block(g, l);
#pragma unroll
            for (int j = 0; j < 32; j++) d[j] ^= v[j];
        }
}

__global__ void __launch_bounds__(BT_THREADS, 2) k_bottom(BottomParams p) {
    extern __shared__ __align__(1024) uint32_t bt_smem[];
    uint32_t* PA = bt_smem;                 // planes of A
    uint32_t* PB = PA + BT_REGION;          // planes of B
    uint32_t* PC = PB + BT_REGION;          // product accumulators
    uint32_t* Pk = PC + BT_REGION;          // per-layer position planes, L x 32
    const int L = p.L;
    // P_k[j] = xor over position bits i (L+i < m) of bit j of s_k(v_(L+i)) * POS_i
    for (int i = threadIdx.x; i < L * 32; i += blockDim.x) {
        const int k = i >> 5, j = i & 31;
        const uint32_t POS[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
        uint32_t v = 0;
        for (int b = 0; b < 5; b++)
            if (L + b < p.m && ((c_S[k * 32 + L + b] >> j) & 1)) v ^= POS[b];
        Pk[i] = v;
    }
    const uint64_t total = p.total;   // loads beyond it read 0, stores beyond it are dropped
    const int lb = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const uint64_t e0 = t << BT_BITS;
        __syncthreads();
        // ---- load + bit-slice both operands (warp = limb, lane = group)
        for (int g = lane; g < BT_GROUPS; g += 32) {
            bt_load_block(p.A, e0, total, g, lb, L, PA);
            bt_load_block(p.B, e0, total, g, lb, L, PB);
        }
        __syncthreads();
        if (p.mode & 1) {
            for (int k = L - 1; k >= 0; k--) {   // FFT_LCH bottom layers, top-down
                bt_layer<false>(PA, k, Pk + k * 32, e0, L, p.m);
                bt_layer<false>(PB, k, Pk + k * 32, e0, L, p.m);
                __syncthreads();
            }
        }
        uint32_t* R = PA;
        if (p.mode & 2) {
            // zero accumulators, then the nine limb products (threads 0..63: one group each)
            for (int i = threadIdx.x; i < BT_REGION; i += blockDim.x) PC[i] = 0;
            __syncthreads();
            if (threadIdx.x < BT_GROUPS) {
                const int g = threadIdx.x;
#pragma unroll 1
                for (int qq = 0; qq < 9; qq++) {
                    uint32_t x[32], y[32], r[32];
                    bt_load_sum(PA, g, c_pm_terms[qq][0], x);
                    bt_load_sum(PB, g, c_pm_terms[qq][0], y);
                    bs_mul32(x, y, r);
                    bt_acc_add(PC, g, c_pm_terms[qq][1], r);
                    if (c_pm_terms[qq][2]) { bs_mul_v31(r, x); bt_acc_add(PC, g, c_pm_terms[qq][2], x); }
                    if (c_pm_terms[qq][3]) { bs_mul_v31sq(r, y); bt_acc_add(PC, g, c_pm_terms[qq][3], y); }
                }
            }
            __syncthreads();
            R = PC;
        }
        if (p.mode & 4) {
            for (int k = 0; k < L; k++) {   // iFFT_LCH bottom layers, bottom-up
                bt_layer<true>(R, k, Pk + k * 32, e0, L, p.m);
                __syncthreads();
            }
        }
        // ---- un-slice and store (A <- R; with mode == 1 also B <- its planes)
        for (int g = lane; g < BT_GROUPS; g += 32) {
            bt_store_block(p.A, e0, total, g, lb, L, R);
            if (p.mode == 1) bt_store_block(p.B, e0, total, g, lb, L, PB);
        }
    }
}

static size_t bottom_smem() { return (size_t)(3 * BT_REGION + 6 * 32) * 4; }
