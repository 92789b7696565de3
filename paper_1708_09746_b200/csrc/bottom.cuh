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

#ifndef BT_TPC
#define BT_TPC 1          // tiles per CTA (2 = one 256-thread CTA per SM whose halves share barriers: measured
#endif                    // phase (one copy of the bs_mul32 code in the instruction caches at a time)
#define BT_HALF 128       // threads per tile
#ifndef BT_PAIR
#define BT_PAIR 0         // 1: forward layers run both operands' products as one paired circuit (bs_mul32x2, the
#endif                    // multiplier's sums shared: 2332 vs 2458 gates) -- measured 9 % slower (spills at 255 regs)
#define BT_THREADS (BT_HALF * BT_TPC)
#define BT_BITS 11
#define BT_GROUPS 64
#define BT_STRIDE 33
#define BT_REGION (4 * BT_GROUPS * BT_STRIDE)   // words per operand region

// pointmul on the planes: the nine TGF(2^32) products of the limb formulas (c_pm_terms in gf2x.cu)
//   R0 = P0 + v31 P1 + v31^2 (P2 + P23)     R1 = P0 + P01 + v31 P23 + v31^2 P3
//   R2 = P0 + v31 P1 + Q0 + v31 Q1          R3 = P0 + P01 + Q0 + Q01
// split over the two threads of a group with the shared parts exchanged through shared memory:
//   h = 0: P3, P1, P0, P01  -> V3 = v31^2 P3 (kept), X2 = P0 + v31 P1, X3 = P0 + P01 (exchanged)
//   h = 1: P23, P2, Q1, Q0, Q01 -> W1 = v31 P23, W0 = v31^2 (P2 + P23) (exchanged), A = Q0 + v31 Q1,
//          B = Q0 + Q01 (kept)
//   then R0 = X2 + W0, R1 = X3 + W1 + V3 (h = 0) and R2 = X2 + A, R3 = X3 + B (h = 1).
// factor limb masks per step (bit l = limb l of the sum a_l, b_l)
__constant__ int c_pm9[2][5] = {{0x8, 0x2, 0x1, 0x3, 0}, {0xC, 0x4, 0xA, 0x5, 0xF}};
#define BT_EX_X2 0
#define BT_EX_X3 1
#define BT_EX_W0 2
#define BT_EX_W1 3

struct BottomParams {
    uint4* A;            // spectrum of a (in: after the direct passes; out: product, after iFFT bottom)
    uint4* B;            // spectrum of b
    uint64_t total;      // batch * N elements per operand (A and B may be adjacent: never touch beyond)
    uint64_t ntiles;     // ceil(total / 2^11)
    int m, L, mode;      // mode bit0: forward layers (A and B), bit1: pointmul (A <- A B), bit2: inverse layers (A)
    IdxMap map;          // local -> global index for the multipliers (identity unless sharded;
                         // the bottom layers and position bits are always below map.pos)
    int l2pf;            // bit 0: thread 0 prefetches the CTA's next tile of A (and B) into L2
};

// (group g of limb lb) -> plane block.  Blocks of groups 32..63 are stored with their low 5 bits
// complemented: the pairs (g0, g0 + 2^k) a warp touches in layer k < 5 are 32 groups spread over both
// halves whose low bits would otherwise coincide pairwise (a 2-way bank conflict on every plane access);
// complementing maps the upper half onto the other 16 banks for every k at once.
__device__ __forceinline__ uint32_t bt_block(int g, int lb) {
    return (uint32_t)((lb * BT_GROUPS + (g ^ ((g & 32) ? 31 : 0))) * BT_STRIDE);
}

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
// U_k(g0) of layer k, pair q: the multiplier of the group's block base with the position bits cleared
__device__ __forceinline__ uint32_t bt_u(int k, int q, uint64_t e0, int L, int m, const IdxMap& map) {
    const int g0 = (q & ((1 << k) - 1)) | ((q >> k) << (k + 1));
    const uint64_t gi = (e0 + bt_elem(g0, 0, L)) & ((1ull << m) - 1);
    return layer_const(k, gidx(map, (uint32_t)gi));
}

// multiplier planes of layer k for this thread's pair: c_j = P_k[j] ^ (bit j of U ? ~0 : 0)
__device__ __forceinline__ uint32_t prmt_sign(uint32_t x, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "r"(sel));
    return r;
}
__device__ __forceinline__ void bt_cplanes(const uint32_t* Pk, uint32_t U, uint32_t* c) {
    // bit j of U replicated over the word: shift it to bit 7 of its byte, then PRMT's sign-replicate mode
    // copies that bit into all four result bytes (selector nibble 8 | byte)
    uint32_t us[8];
#pragma unroll
    for (int k = 0; k < 8; k++) us[k] = U << k;
#pragma unroll
    for (int j = 0; j < 32; j++) c[j] = Pk[j] ^ prmt_sign(us[7 - (j & 7)], (8u | (uint32_t)(j >> 3)) * 0x1111u);
}

// x * c for 32 bit-sliced TGF(2^32) elements x and multiplier planes c whose planes >= W are zero (the layer's
// multipliers are < 2^W, multiplier shortening P:802-815): for W = 8 / 16 each 8- / 16-bit block of x is
// multiplied by c on its own (Prop. 2) -- 4 x 110 / 2 x 375 gates instead of 1229
template <int W>
__device__ __forceinline__ void bs_mul_w(const uint32_t* x, const uint32_t* c, uint32_t* r) {
    if (W == 8) { bs_mul8(x, c, r); bs_mul8(x + 8, c, r + 8); bs_mul8(x + 16, c, r + 16); bs_mul8(x + 24, c, r + 24); }
    else if (W == 16) { bs_mul16(x, c, r); bs_mul16(x + 16, c, r + 16); }
    else bs_mul32(x, c, r);
}

// CK: cache of the multiplier planes, [layer][pair][33] (written by warp 0 in the forward layers,
// read by every warp in the inverse layers of the same tile)
template <bool INV, int W = 32>
__device__ __forceinline__ void bt_layer(uint32_t* planes, int k, const uint32_t* Pk, const uint32_t* UC,
                                         uint32_t* CK, int tid) {
    const int lb = tid >> 5, q = tid & 31;
    const int g0 = (q & ((1 << k) - 1)) | ((q >> k) << (k + 1));
    const int g1 = g0 | (1 << k);
    uint32_t c[32], x1[32], pr[32];
    if (CK) {
        const uint32_t* ck = CK + (k * 32 + q) * 33;
#pragma unroll
        for (int j = 0; j < 32; j++) c[j] = ck[j];
    } else {
        bt_cplanes(Pk, UC[k * 32 + q], c);
    }
    uint32_t* b0 = planes + bt_block(g0, lb);
    uint32_t* b1 = planes + bt_block(g1, lb);
#pragma unroll
    for (int j = 0; j < 32; j++) x1[j] = b1[j];
    if (INV) {
#pragma unroll
        for (int j = 0; j < 32; j++) x1[j] ^= b0[j];
    }
    bs_mul_w<W>(x1, c, pr);
#pragma unroll
    for (int j = 0; j < 32; j++) {
        const uint32_t x0 = b0[j] ^ pr[j];
        b0[j] = x0;
        b1[j] = INV ? x1[j] : (x1[j] ^ x0);
    }
}

// forward layer k on both operands with one set of multiplier planes (stored to CK by warp 0)
template <int W = 32>
__device__ __forceinline__ void bt_layer2(uint32_t* PA, uint32_t* PB, int k, const uint32_t* Pk, const uint32_t* UC,
                                          uint32_t* CK, int tid) {
    const int lb = tid >> 5, q = tid & 31;
    const int g0 = (q & ((1 << k) - 1)) | ((q >> k) << (k + 1));
    const int g1 = g0 | (1 << k);
    uint32_t c[32], x1[32], pr[32];
    bt_cplanes(Pk, UC[k * 32 + q], c);
    if (CK && lb == 0) {
        uint32_t* ck = CK + (k * 32 + q) * 33;
#pragma unroll
        for (int j = 0; j < 32; j++) ck[j] = c[j];
    }
    if (W == 32 && BT_PAIR) {
        // both operands' products in one generated circuit (bs_mul32x2): the multiplier's Karatsuba sums once,
        // two independent instruction streams
        uint32_t y1[32], qr[32];
        uint32_t* a0p = PA + bt_block(g0, lb);
        uint32_t* a1p = PA + bt_block(g1, lb);
        uint32_t* b0p = PB + bt_block(g0, lb);
        uint32_t* b1p = PB + bt_block(g1, lb);
#pragma unroll
        for (int j = 0; j < 32; j++) { x1[j] = a1p[j]; y1[j] = b1p[j]; }
        bs_mul32x2(x1, y1, c, pr, qr);
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const uint32_t x0 = a0p[j] ^ pr[j];
            a0p[j] = x0;
            a1p[j] = x1[j] ^ x0;
            const uint32_t y0 = b0p[j] ^ qr[j];
            b0p[j] = y0;
            b1p[j] = y1[j] ^ y0;
        }
        return;
    }
#pragma unroll 1
    for (int o = 0; o < 2; o++) {
        uint32_t* planes = o ? PB : PA;
        uint32_t* b0 = planes + bt_block(g0, lb);
        uint32_t* b1 = planes + bt_block(g1, lb);
#pragma unroll
        for (int j = 0; j < 32; j++) x1[j] = b1[j];
        bs_mul_w<W>(x1, c, pr);
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const uint32_t x0 = b0[j] ^ pr[j];
            b0[j] = x0;
            b1[j] = x1[j] ^ x0;
        }
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

// SUBW: some layer's multipliers lie below 2^16 (small transforms): per-layer width dispatch to bs_mul_w (a
// separate instantiation: compiled into the plain kernel the dispatch cost the headline c4b 2 %)
template <bool SUBW>
__global__ void __launch_bounds__(BT_THREADS, 2 / BT_TPC) k_bottom(BottomParams p) {
    extern __shared__ __align__(1024) uint32_t bt_smem[];
    const int half = BT_TPC == 1 ? 0 : (int)(threadIdx.x / BT_HALF), tid = threadIdx.x % BT_HALF;
    uint32_t* PA = bt_smem + half * 2 * BT_REGION;   // planes of A (this half's tile)
    uint32_t* PB = PA + BT_REGION;                   // planes of B
    uint32_t* Pk = bt_smem + BT_TPC * 2 * BT_REGION; // per-layer position planes, L x 32 (shared)
    uint32_t* UCb = Pk + 6 * 32;                     // per tile: U_k of each (layer, pair), BT_TPC x 6 x 32
    uint32_t* UC = UCb + half * 6 * 32;
    uint32_t* EX = UCb + BT_TPC * 6 * 32 + half * 4 * 64 * 33;   // pointmul exchange sets, 4 x 64 x 33
    uint32_t* CK = nullptr;   // (a multiplier-plane cache for the inverse layers measured +0.5 %: the space holds EX)
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
    const int lb = tid >> 5, lane = tid & 31;
    // both halves iterate together (shared barriers); a half past the last tile loads zeros and
    // drops its stores (e0 >= total)
    for (uint64_t tb = (uint64_t)blockIdx.x * BT_TPC; tb < p.ntiles; tb += (uint64_t)gridDim.x * BT_TPC) {
        const uint64_t e0 = (tb + half) << BT_BITS;
        if ((p.l2pf & 1) && tid == 0) {   // the CTA's next tile(s) into L2 while this one runs
            const uint64_t n0 = (tb + (uint64_t)gridDim.x * BT_TPC) << BT_BITS;
            if (n0 + ((uint64_t)BT_TPC << BT_BITS) <= total) {
                bulk_prefetch_l2(p.A + n0, (uint32_t)(16u << BT_BITS) * BT_TPC);
                if (p.mode & 3) bulk_prefetch_l2(p.B + n0, (uint32_t)(16u << BT_BITS) * BT_TPC);
            }
        }
        __syncthreads();
        for (int i = tid; i < L * 32; i += BT_HALF) UC[i] = bt_u(i >> 5, i & 31, e0, L, p.m, p.map);
        // ---- load + bit-slice both operands (warp = limb, lane = group)
        // (one rolled loop: this straight-line code runs once per tile and would otherwise miss the
        // instruction caches on every copy)
        const int nld = (p.mode & 3) ? 2 : 1;   // inverse-only tiles (mode 4) need no B
#pragma unroll 1
        for (int it = 0; it < nld * BT_GROUPS / 32; it++) {
            const int g = lane + 32 * (nld == 2 ? (it >> 1) : it);
            const bool isb = nld == 2 && (it & 1);
            bt_load_block(isb ? p.B : p.A, e0, total, g, lb, L, isb ? PB : PA);
        }
        __syncthreads();
        if (p.mode & 1) {
            // FFT_LCH bottom layers, top-down; one set of multiplier planes per layer serves both operands
#pragma unroll 1
            for (int k = L - 1; k >= 0; k--) {
                const int wc = p.m + p.map.bits - k;   // the layer's multipliers are < 2^wc
                if (SUBW && wc <= 8) bt_layer2<8>(PA, PB, k, Pk + k * 32, UC, CK, tid);
                else if (SUBW && wc <= 16) bt_layer2<16>(PA, PB, k, Pk + k * 32, UC, CK, tid);
                else bt_layer2<32>(PA, PB, k, Pk + k * 32, UC, CK, tid);
                __syncthreads();
            }
        }
        uint32_t* R = PA;
        if (p.mode & 2) {
            const int g = tid & (BT_GROUPS - 1), h = tid >> 6;
            uint32_t* ex = EX + g * 33;   // exchange set e of group g at ex + e * 64 * 33
            uint32_t a0[32], a1[32];
#pragma unroll 1
            for (int st = 0; st < 4 + h; st++) {
                uint32_t x[32], y[32], r[32];
                const int mask = c_pm9[h][st];
                bt_load_sum(PA, g, mask, x);
                bt_load_sum(PB, g, mask, y);
                bs_mul32(x, y, r);
                switch (h * 5 + st) {
                    case 0: bs_mul_v31sq(r, a0); break;                                   // V3
                    case 1: bs_mul_v31(r, a1); break;                                     // v31 P1
                    case 2:                                                               // X2, then P0
#pragma unroll
                        for (int j = 0; j < 32; j++) { ex[BT_EX_X2 * 64 * 33 + j] = a1[j] ^ r[j]; a1[j] = r[j]; }
                        break;
                    case 3:                                                               // X3
#pragma unroll
                        for (int j = 0; j < 32; j++) ex[BT_EX_X3 * 64 * 33 + j] = a1[j] ^ r[j];
                        break;
                    case 5:                                                               // P23, W1
                        bs_mul_v31(r, x);
#pragma unroll
                        for (int j = 0; j < 32; j++) { a1[j] = r[j]; ex[BT_EX_W1 * 64 * 33 + j] = x[j]; }
                        break;
                    case 6:                                                               // W0
#pragma unroll
                        for (int j = 0; j < 32; j++) a1[j] ^= r[j];
                        bs_mul_v31sq(a1, y);
#pragma unroll
                        for (int j = 0; j < 32; j++) ex[BT_EX_W0 * 64 * 33 + j] = y[j];
                        break;
                    case 7: bs_mul_v31(r, a0); break;                                     // v31 Q1
                    case 8:                                                               // A, B = Q0
#pragma unroll
                        for (int j = 0; j < 32; j++) { a0[j] ^= r[j]; a1[j] = r[j]; }
                        break;
                    default:                                                              // B += Q01
#pragma unroll
                        for (int j = 0; j < 32; j++) a1[j] ^= r[j];
                        break;
                }
            }
            __syncthreads();   // A and B planes read, exchange sets written
            uint32_t* d0 = PA + bt_block(g, 2 * h);
            uint32_t* d1 = PA + bt_block(g, 2 * h + 1);
            if (h == 0) {
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    d0[j] = ex[BT_EX_X2 * 64 * 33 + j] ^ ex[BT_EX_W0 * 64 * 33 + j];
                    d1[j] = ex[BT_EX_X3 * 64 * 33 + j] ^ ex[BT_EX_W1 * 64 * 33 + j] ^ a0[j];
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    d0[j] = ex[BT_EX_X2 * 64 * 33 + j] ^ a0[j];
                    d1[j] = ex[BT_EX_X3 * 64 * 33 + j] ^ a1[j];
                }
            }
            __syncthreads();
        }
        if (p.mode & 4) {
            for (int k = 0; k < L; k++) {   // iFFT_LCH bottom layers, bottom-up
                const int wc = p.m + p.map.bits - k;
                if (SUBW && wc <= 8) bt_layer<true, 8>(R, k, Pk + k * 32, UC, CK, tid);
                else if (SUBW && wc <= 16) bt_layer<true, 16>(R, k, Pk + k * 32, UC, CK, tid);
                else bt_layer<true, 32>(R, k, Pk + k * 32, UC, CK, tid);
                __syncthreads();
            }
        }
        // ---- un-slice and store (A <- R; with mode == 1 also B <- its planes)
        const int nst = (p.mode == 1 ? 2 : 1) * BT_GROUPS / 32;
#pragma unroll 1
        for (int it = 0; it < nst; it++) {
            const int g = lane + 32 * (it & 1);
            bt_store_block((it & 2) ? p.B : p.A, e0, total, g, lb, L, (it & 2) ? PB : R);
        }
    }
}

static size_t bottom_smem() { return (size_t)(BT_TPC * 2 * BT_REGION + 6 * 32 + BT_TPC * (6 * 32 + 4 * 64 * 33)) * 4; }

static int grid_for(uint64_t items, int per_block, int sm_count, int occ);
static int bottom_l2pf();
static void bottom_launch(const BottomParams& bp, int smc, cudaStream_t st) {
    const bool subw = bp.m + bp.map.bits - (bp.L - 1) <= 16;   // the lowest layer's multipliers are < 2^16
    const int g = grid_for((bp.ntiles + BT_TPC - 1) / BT_TPC, 1, smc, 2 / BT_TPC);
    BottomParams q = bp;
    q.l2pf = bottom_l2pf();
    if (subw) k_bottom<true><<<g, BT_THREADS, bottom_smem(), st>>>(q);
    else k_bottom<false><<<g, BT_THREADS, bottom_smem(), st>>>(q);
}
