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

// pointmul split by output limbs (limb formulas: see c_pm_terms in gf2x.cu).  Per half h, six
// products {factor limb mask, gets r, gets v31 r, gets v31^2 r}; bit 0 = first limb of the half
// (R0 / R2), bit 1 = second (R1 / R3).
//   R0 = P0 + v31 P1 + v31^2 (P2 + P23)        R1 = P0 + P01 + v31 P23 + v31^2 P3
//   R2 = P0 + Q0 + v31 (P1 + Q1)               R3 = P0 + P01 + Q0 + Q01
__constant__ int c_pm_half[2][6][4] = {
    {{0x1, 0x3, 0x0, 0x0},    // P0  -> R0 R1
     {0x2, 0x0, 0x1, 0x0},    // P1  -> v31: R0
     {0x4, 0x0, 0x0, 0x1},    // P2  -> v31^2: R0
     {0xC, 0x0, 0x2, 0x1},    // P23 -> v31: R1, v31^2: R0
     {0x3, 0x2, 0x0, 0x0},    // P01 -> R1
     {0x8, 0x0, 0x0, 0x2}},   // P3  -> v31^2: R1
    {{0x1, 0x3, 0x0, 0x0},    // P0  -> R2 R3
     {0x5, 0x3, 0x0, 0x0},    // Q0  -> R2 R3
     {0x2, 0x0, 0x1, 0x0},    // P1  -> v31: R2
     {0xA, 0x0, 0x1, 0x0},    // Q1  -> v31: R2
     {0x3, 0x2, 0x0, 0x0},    // P01 -> R3
     {0xF, 0x2, 0x0, 0x0}},   // Q01 -> R3
};

struct BottomParams {
    uint4* A;            // spectrum of a (in: after the direct passes; out: product, after iFFT bottom)
    uint4* B;            // spectrum of b
    uint64_t total;      // batch * N elements per operand (A and B may be adjacent: never touch beyond)
    uint64_t ntiles;     // ceil(total / 2^11)
    int m, L, mode;      // mode bit0: forward layers, bit1: pointmul, bit2: inverse layers
    IdxMap map;          // local -> global index for the multipliers (identity unless sharded;
                         // the bottom layers and position bits are always below map.pos)
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
__device__ __forceinline__ void bt_layer(uint32_t* planes, int k, const uint32_t* Pk, uint64_t e0, int L, int m,
                                         const IdxMap& map) {
    const int lb = threadIdx.x >> 5, q = threadIdx.x & 31;
    const int g0 = (q & ((1 << k) - 1)) | ((q >> k) << (k + 1));
    const int g1 = g0 | (1 << k);
    // U_k(g0): within-pair index of the group's block base with the position bits cleared
    const uint64_t N = 1ull << m;
    const uint64_t gi = (e0 + bt_elem(g0, 0, L)) & (N - 1);
    const uint32_t U = layer_const(k, gidx(map, (uint32_t)gi));
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
    uint32_t* Pk = PB + BT_REGION;          // per-layer position planes, L x 32
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
                bt_layer<false>(PA, k, Pk + k * 32, e0, L, p.m, p.map);
                bt_layer<false>(PB, k, Pk + k * 32, e0, L, p.m, p.map);
                __syncthreads();
            }
        }
        uint32_t* R = PA;
        if (p.mode & 2) {
            // two threads per group: thread h = 0 produces result limbs R0, R1, h = 1 produces R2, R3
            // (six TGF(2^32) products each, accumulated in registers), then both overwrite the A planes
            const int g = threadIdx.x & (BT_GROUPS - 1), h = threadIdx.x >> 6;
            uint32_t acc0[32], acc1[32];
#pragma unroll
            for (int j = 0; j < 32; j++) { acc0[j] = 0; acc1[j] = 0; }
#pragma unroll 1
            for (int qq = 0; qq < 6; qq++) {
                const int* T = c_pm_half[h][qq];
                uint32_t x[32], y[32], r[32];
                bt_load_sum(PA, g, T[0], x);
                bt_load_sum(PB, g, T[0], y);
                bs_mul32(x, y, r);
                // T[1..3]: which of the two output limbs get r, v31 r, v31^2 r (bit 0: first, bit 1: second)
                if (T[2]) bs_mul_v31(r, x);
                if (T[3]) bs_mul_v31sq(r, y);
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    uint32_t a0 = acc0[j], a1 = acc1[j];
                    if (T[1] & 1) a0 ^= r[j];
                    if (T[1] & 2) a1 ^= r[j];
                    if (T[2] & 1) a0 ^= x[j];
                    if (T[2] & 2) a1 ^= x[j];
                    if (T[3] & 1) a0 ^= y[j];
                    if (T[3] & 2) a1 ^= y[j];
                    acc0[j] = a0; acc1[j] = a1;
                }
            }
            __syncthreads();   // every thread is done reading A and B
            uint32_t* d0 = PA + bt_block(g, 2 * h);
            uint32_t* d1 = PA + bt_block(g, 2 * h + 1);
#pragma unroll
            for (int j = 0; j < 32; j++) { d0[j] = acc0[j]; d1[j] = acc1[j]; }
            __syncthreads();
        }
        if (p.mode & 4) {
            for (int k = 0; k < L; k++) {   // iFFT_LCH bottom layers, bottom-up
                bt_layer<true>(R, k, Pk + k * 32, e0, L, p.m, p.map);
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

static size_t bottom_smem() { return (size_t)(2 * BT_REGION + 6 * 32) * 4; }
