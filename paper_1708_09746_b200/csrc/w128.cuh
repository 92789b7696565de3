// w128.cuh -- Alg. 5 with 128-bit blocks over TGF(2^256) ("An initial block width
// of w=128 bits is also possible and in this case the operative field is TGF(2^256)"; sec 4.2
// P:1077-1114).  Included by gf2x.cu after the w = 64 pipeline.
//
// TGF(2^256) = TGF(2^128)[x_8]/(x_8^2 + x_8 + v_127) (the tower of P:640-652 one level up).  A spectrum
// of N elements is stored as two planes of N uint4: the low halves (coordinates of v_0..v_127) and the
// high halves (coefficient of x_8).  Every FFT multiplier s_k(phi_v(b)) lies in TGF(2^32), and by
// Prop. 2 a subfield constant multiplies the two halves independently, so FFT_LCH over
// TGF(2^256) is the w = 64 FFT kernels applied to both planes (the planes are "products" of the batch
// with identical multipliers); likewise the XOR-only BasisCvt/iBasisCvt.  What is new:
//   k_psi256_bs   changeRepr 128-bit polynomial-basis block -> TGF(2^256), bit-sliced generated networks
//                 (k_psi256: M4R-4 tables, for N < 2048)
//   k_w128_sums   a_lo + a_hi, b_lo + b_hi (Karatsuba operands)
//   k_bottom x3   mode 2: the three TGF(2^128) products P0 = a_lo b_lo, P2 = a_hi b_hi,
//                 P1 = (a_lo + a_hi)(b_lo + b_hi), bit-sliced (the w = 64 pointmul)
//   k_w128_post   lo = P0 + v_127 P2, hi = P1 + P0 (Karatsuba at the x_8 level, sec 4.1.3)
//   k_ipsi256_bs  changeRepr^-1 to the 256-bit polynomial basis + InterleavedCombine on 128-bit blocks,
//                 bit-sliced (k_ipsi256: M4R-4, for N < 2048 or ragged output lengths)
// Plane layout per operand: [lo planes of all batch products][hi planes], so each plane set is one
// contiguous run for the bottom kernel.
#pragma once

struct DevTables256 {
    uint4 psi[32 * 16 * 2];    // M4R-4: nibble t of a 128-bit block, value x -> image (lo, hi) in the tower
    uint4 ipsi[64 * 16 * 2];   // M4R-4: nibble t of a tower element (t < 32: lo half), x -> polynomial (lo, hi)
    uint4 v127[16 * 256];      // M4R-8: byte ch of a TGF(2^128) element, x -> v_127 (x) (x << 8 ch)
};

static void host_build_tables256(DevTables256* T) {
    using namespace gf2x_host;
    static Isomorphism256 iso;
    build_isomorphism256(&iso);
    auto put = [](uint4* d, const W256& v) {
        d[0] = make_uint4((uint32_t)v.w[0], (uint32_t)(v.w[0] >> 32), (uint32_t)v.w[1], (uint32_t)(v.w[1] >> 32));
        d[1] = make_uint4((uint32_t)v.w[2], (uint32_t)(v.w[2] >> 32), (uint32_t)v.w[3], (uint32_t)(v.w[3] >> 32));
    };
    for (int t = 0; t < 32; t++)
        for (int x = 0; x < 16; x++) {
            W256 v = w256_zero();
            for (int b = 0; b < 4; b++)
                if ((x >> b) & 1) w256_xor(v, iso.polyToTower[4 * t + b]);
            put(&T->psi[(t * 16 + x) * 2], v);
        }
    for (int t = 0; t < 64; t++)
        for (int x = 0; x < 16; x++) {
            W256 v = w256_zero();
            for (int b = 0; b < 4; b++)
                if ((x >> b) & 1) w256_xor(v, iso.towerToPoly[4 * t + b]);
            put(&T->ipsi[(t * 16 + x) * 2], v);
        }
    const u128 v127 = ((u128)1) << 127;
    for (int ch = 0; ch < 16; ch++)
        for (int x = 0; x < 256; x++) {
            const u128 r = tower_mul(((u128)x) << (8 * ch), v127);
            T->v127[ch * 256 + x] = make_uint4((uint32_t)r, (uint32_t)(r >> 32), (uint32_t)(r >> 64), (uint32_t)(r >> 96));
        }
}

// ---------------------------------------------------------------------------------------------
// changeRepr: element i of operand o, product p: the 128-bit block S[o][p][i] (i < s_per,
// 0 beyond) -> planes W[o][lo/hi][p][i].  One thread per element, 32 nibble lookups of 32 B.
// ---------------------------------------------------------------------------------------------
#define PSI256_THREADS 256
__global__ void __launch_bounds__(PSI256_THREADS) k_psi256(const uint4* __restrict__ S, uint64_t s_per, uint64_t N,
                                                           uint64_t batch, int ops, const DevTables256* __restrict__ T,
                                                           uint4* __restrict__ W) {
    __shared__ uint4 tab[32 * 16 * 2];
    for (int i = threadIdx.x; i < 32 * 16 * 2; i += blockDim.x) tab[i] = T->psi[i];
    __syncthreads();
    const uint64_t per_op = batch * N, total = per_op * ops;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = e / per_op, r = e - o * per_op, p = r / N, i = r - p * N;
        uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
        if (i < s_per) {
            const uint4 x = S[(o * batch + p) * s_per + i];
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int L = 0; L < 4; L++) {
                if (!w[L]) continue;
#pragma unroll
                for (int n = 0; n < 8; n++) {
                    const uint32_t t = L * 8 + n, v = (w[L] >> (4 * n)) & 15;
                    lo = xor4(lo, tab[(t * 16 + v) * 2]);
                    hi = xor4(hi, tab[(t * 16 + v) * 2 + 1]);
                }
            }
        }
        uint4* d = W + o * 2 * per_op + p * N + i;
        d[0] = lo;
        d[per_op] = hi;
    }
}

// Karatsuba operands: Ts = lo + hi for n elements (lo plane at P, hi plane at P + n)
__global__ void k_w128_sums(const uint4* __restrict__ P, uint64_t n, uint4* __restrict__ Ts) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        Ts[i] = xor4(P[i], P[n + i]);
}

// x_8-level recombination: with P0 in the lo plane, P2 in the hi plane, P1 in Ts:
//   lo = P0 + v_127 (x) P2,  hi = P1 + P0.   v_127 (x) P2 by M4R-8 (16 byte lookups).
__global__ void __launch_bounds__(256) k_w128_post(uint4* __restrict__ P, uint64_t n, const uint4* __restrict__ Ts,
                                                   const DevTables256* __restrict__ T) {
    extern __shared__ uint4 v127t[];   // 16 x 256
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) v127t[i] = T->v127[i];
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 p0 = P[i], p2 = P[n + i], p1 = Ts[i];
        const uint32_t w[4] = {p2.x, p2.y, p2.z, p2.w};
        uint4 lo = p0;
#pragma unroll
        for (int L = 0; L < 4; L++)
#pragma unroll
            for (int b = 0; b < 4; b++) lo = xor4(lo, v127t[(L * 4 + b) * 256 + ((w[L] >> (8 * b)) & 255)]);
        P[i] = lo;
        P[n + i] = xor4(p1, p0);
    }
}

// ---------------------------------------------------------------------------------------------
// changeRepr^-1 + InterleavedCombine on 128-bit blocks:
//   C_i = psi256^-1(lo_i, hi_i) (degree <= 254), out block w = lo128(C_w) ^ hi128(C_(w-1)),
// words 2w, 2w+1 of the product, w < ceil(n_out / 2) (C_i = 0 for i >= N).  A CTA covers 256 blocks
// of one product; thread 0 also converts the element before the CTA's first block.
// ---------------------------------------------------------------------------------------------
#define IPSI256_THREADS 256
__device__ __forceinline__ void ipsi256_apply(const uint4* tab, uint4 lo, uint4 hi, uint4& rlo, uint4& rhi) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    rlo = make_uint4(0, 0, 0, 0);
    rhi = rlo;
#pragma unroll
    for (int L = 0; L < 8; L++) {
        if (!w[L]) continue;
#pragma unroll
        for (int n = 0; n < 8; n++) {
            const uint32_t t = L * 8 + n, v = (w[L] >> (4 * n)) & 15;
            rlo = xor4(rlo, tab[(t * 16 + v) * 2]);
            rhi = xor4(rhi, tab[(t * 16 + v) * 2 + 1]);
        }
    }
}
__global__ void __launch_bounds__(IPSI256_THREADS) k_ipsi256(const uint4* __restrict__ W, uint64_t N, uint64_t batch,
                                                             uint64_t n_out, const DevTables256* __restrict__ T,
                                                             uint64_t* __restrict__ out) {
    extern __shared__ uint4 ib_tab[];   // 64 x 16 x 2 (32 KB)
    __shared__ uint4 Hs[IPSI256_THREADS + 1];
    for (int i = threadIdx.x; i < 64 * 16 * 2; i += blockDim.x) ib_tab[i] = T->ipsi[i];
    const uint64_t nblk = (n_out + 1) / 2;
    const uint64_t cta_per = (nblk + IPSI256_THREADS - 1) / IPSI256_THREADS;
    const uint64_t plane = N * batch;
    for (uint64_t cb = blockIdx.x; cb < cta_per * batch; cb += gridDim.x) {
        const uint64_t p = cb / cta_per, w0 = (cb - p * cta_per) * IPSI256_THREADS;
        const uint4* lo = W + p * N;
        const uint4* hi = lo + plane;
        __syncthreads();   // tables loaded / previous tile's Hs consumed
        const uint64_t w = w0 + threadIdx.x;
        uint4 clo = make_uint4(0, 0, 0, 0), chi = clo;
        if (w < nblk && w < N) ipsi256_apply(ib_tab, lo[w], hi[w], clo, chi);
        Hs[threadIdx.x + 1] = chi;
        if (threadIdx.x == 0) {
            uint4 plo = make_uint4(0, 0, 0, 0), phi = plo;
            if (w0 >= 1 && w0 - 1 < N) ipsi256_apply(ib_tab, lo[w0 - 1], hi[w0 - 1], plo, phi);
            Hs[0] = phi;
        }
        __syncthreads();
        if (w < nblk) {
            const uint4 v = xor4(clo, Hs[threadIdx.x]);
            uint64_t* d = out + p * n_out + 2 * w;
            d[0] = ((uint64_t)v.y << 32) | v.x;
            if (2 * w + 1 < n_out) d[1] = ((uint64_t)v.w << 32) | v.z;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Bit-sliced changeRepr / changeRepr^-1 for w = 128 (generated XOR networks of the same isomorphism,
// tools/gen_bitslice.py + tools/dump_iso.cpp): a thread owns 32 consecutive elements of a 2048-element
// tile, transposes each 32-bit limb into 32 planes (plane j = bit j of the 32 limbs) and runs the
// 32 x 32 blocks of the map; output limbs are produced two at a time, transposed back and staged in
// shared memory for the stores.  Tiles never straddle products (N % W2_TILE == 0).
// ---------------------------------------------------------------------------------------------
#define W2_THREADS 64
#define W2_TILE (32 * W2_THREADS)
__device__ __forceinline__ uint32_t w2_swz(uint32_t e) { return e ^ ((e >> 5) & 31); }

// acc pair (a0, a1) = output limbs (O, O + 1) of changeRepr_256 from the 4 input limbs' planes
__device__ __forceinline__ void psi256_block(int O, int L, const uint32_t* x, uint32_t* a0, uint32_t* a1) {
    switch (O * 4 + L) {
        case 0: bs_psi256_0_0(x, a0); bs_psi256_1_0(x, a1); break;
        case 1: bs_psi256_0_1(x, a0); bs_psi256_1_1(x, a1); break;
        case 2: bs_psi256_0_2(x, a0); bs_psi256_1_2(x, a1); break;
        case 3: bs_psi256_0_3(x, a0); bs_psi256_1_3(x, a1); break;
        case 8: bs_psi256_2_0(x, a0); bs_psi256_3_0(x, a1); break;
        case 9: bs_psi256_2_1(x, a0); bs_psi256_3_1(x, a1); break;
        case 10: bs_psi256_2_2(x, a0); bs_psi256_3_2(x, a1); break;
        case 11: bs_psi256_2_3(x, a0); bs_psi256_3_3(x, a1); break;
        case 16: bs_psi256_4_0(x, a0); bs_psi256_5_0(x, a1); break;
        case 17: bs_psi256_4_1(x, a0); bs_psi256_5_1(x, a1); break;
        case 18: bs_psi256_4_2(x, a0); bs_psi256_5_2(x, a1); break;
        case 19: bs_psi256_4_3(x, a0); bs_psi256_5_3(x, a1); break;
        case 24: bs_psi256_6_0(x, a0); bs_psi256_7_0(x, a1); break;
        case 25: bs_psi256_6_1(x, a0); bs_psi256_7_1(x, a1); break;
        case 26: bs_psi256_6_2(x, a0); bs_psi256_7_2(x, a1); break;
        case 27: bs_psi256_6_3(x, a0); bs_psi256_7_3(x, a1); break;
    }
}
__device__ __forceinline__ void ipsi256_block(int O, int L, const uint32_t* x, uint32_t* a0, uint32_t* a1) {
    switch (O * 8 + L) {
        case 0: bs_ipsi256_0_0(x, a0); bs_ipsi256_1_0(x, a1); break;
        case 1: bs_ipsi256_0_1(x, a0); bs_ipsi256_1_1(x, a1); break;
        case 2: bs_ipsi256_0_2(x, a0); bs_ipsi256_1_2(x, a1); break;
        case 3: bs_ipsi256_0_3(x, a0); bs_ipsi256_1_3(x, a1); break;
        case 4: bs_ipsi256_0_4(x, a0); bs_ipsi256_1_4(x, a1); break;
        case 5: bs_ipsi256_0_5(x, a0); bs_ipsi256_1_5(x, a1); break;
        case 6: bs_ipsi256_0_6(x, a0); bs_ipsi256_1_6(x, a1); break;
        case 7: bs_ipsi256_0_7(x, a0); bs_ipsi256_1_7(x, a1); break;
        case 16: bs_ipsi256_2_0(x, a0); bs_ipsi256_3_0(x, a1); break;
        case 17: bs_ipsi256_2_1(x, a0); bs_ipsi256_3_1(x, a1); break;
        case 18: bs_ipsi256_2_2(x, a0); bs_ipsi256_3_2(x, a1); break;
        case 19: bs_ipsi256_2_3(x, a0); bs_ipsi256_3_3(x, a1); break;
        case 20: bs_ipsi256_2_4(x, a0); bs_ipsi256_3_4(x, a1); break;
        case 21: bs_ipsi256_2_5(x, a0); bs_ipsi256_3_5(x, a1); break;
        case 22: bs_ipsi256_2_6(x, a0); bs_ipsi256_3_6(x, a1); break;
        case 23: bs_ipsi256_2_7(x, a0); bs_ipsi256_3_7(x, a1); break;
        case 32: bs_ipsi256_4_0(x, a0); bs_ipsi256_5_0(x, a1); break;
        case 33: bs_ipsi256_4_1(x, a0); bs_ipsi256_5_1(x, a1); break;
        case 34: bs_ipsi256_4_2(x, a0); bs_ipsi256_5_2(x, a1); break;
        case 35: bs_ipsi256_4_3(x, a0); bs_ipsi256_5_3(x, a1); break;
        case 36: bs_ipsi256_4_4(x, a0); bs_ipsi256_5_4(x, a1); break;
        case 37: bs_ipsi256_4_5(x, a0); bs_ipsi256_5_5(x, a1); break;
        case 38: bs_ipsi256_4_6(x, a0); bs_ipsi256_5_6(x, a1); break;
        case 39: bs_ipsi256_4_7(x, a0); bs_ipsi256_5_7(x, a1); break;
        case 48: bs_ipsi256_6_0(x, a0); bs_ipsi256_7_0(x, a1); break;
        case 49: bs_ipsi256_6_1(x, a0); bs_ipsi256_7_1(x, a1); break;
        case 50: bs_ipsi256_6_2(x, a0); bs_ipsi256_7_2(x, a1); break;
        case 51: bs_ipsi256_6_3(x, a0); bs_ipsi256_7_3(x, a1); break;
        case 52: bs_ipsi256_6_4(x, a0); bs_ipsi256_7_4(x, a1); break;
        case 53: bs_ipsi256_6_5(x, a0); bs_ipsi256_7_5(x, a1); break;
        case 54: bs_ipsi256_6_6(x, a0); bs_ipsi256_7_6(x, a1); break;
        case 55: bs_ipsi256_6_7(x, a0); bs_ipsi256_7_7(x, a1); break;
    }
}

// thread-own planes of input limb L -> x (in place transposed data in In)
__device__ __forceinline__ void w2_load_planes(const uint32_t* In, int L, uint32_t e0, uint32_t* x) {
#pragma unroll
    for (int j = 0; j < 32; j++) x[j] = In[L * W2_TILE + w2_swz(e0 + j)];
}
__device__ __forceinline__ void w2_transpose_own(uint32_t* In, int nl, uint32_t e0) {
#pragma unroll 1
    for (int L = 0; L < nl; L++) {
        uint32_t x[32];
        w2_load_planes(In, L, e0, x);
        transpose32(x);
#pragma unroll
        for (int j = 0; j < 32; j++) In[L * W2_TILE + w2_swz(e0 + j)] = x[j];
    }
}

// changeRepr: S[(o batch + p) s_per + i] (0 for i >= s_per) -> W[o][lo/hi plane][p][i]
__global__ void __launch_bounds__(W2_THREADS) k_psi256_bs(const uint4* __restrict__ S, uint64_t s_per, uint64_t N,
                                                          uint64_t batch, int ops, uint4* __restrict__ W) {
    extern __shared__ __align__(1024) uint32_t w2_smem[];
    uint32_t* In = w2_smem;                  // [4][W2_TILE] limb planes
    uint32_t* Stg = w2_smem + 4 * W2_TILE;   // [2][W2_TILE] two output limbs
    const uint64_t per_op = batch * N, ntiles = per_op * ops / W2_TILE;
    const uint32_t t = threadIdx.x, e0 = 32 * t;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t g0 = tile * W2_TILE, o = g0 / per_op, r0 = g0 - o * per_op, p = r0 / N, i0 = r0 - p * N;
        const uint4* src = S + (o * batch + p) * s_per;
        __syncthreads();   // previous tile's stores done with Stg / In
        for (uint32_t e = t; e < W2_TILE; e += W2_THREADS) {
            const uint64_t i = i0 + e;
            const uint4 v = i < s_per ? src[i] : make_uint4(0, 0, 0, 0);
            const uint32_t q = w2_swz(e);
            In[q] = v.x; In[W2_TILE + q] = v.y; In[2 * W2_TILE + q] = v.z; In[3 * W2_TILE + q] = v.w;
        }
        __syncthreads();
        w2_transpose_own(In, 4, e0);
        uint4* dlo = W + o * 2 * per_op + p * N + i0;
#pragma unroll 1
        for (int O = 0; O < 8; O += 2) {
            uint32_t a0[32], a1[32];
#pragma unroll
            for (int j = 0; j < 32; j++) { a0[j] = 0; a1[j] = 0; }
#pragma unroll 1
            for (int L = 0; L < 4; L++) {
                uint32_t x[32];
                w2_load_planes(In, L, e0, x);
                psi256_block(O, L, x, a0, a1);
            }
            transpose32(a0);
            transpose32(a1);
            __syncthreads();   // previous pair's stores have read Stg
#pragma unroll
            for (int j = 0; j < 32; j++) { Stg[w2_swz(e0 + j)] = a0[j]; Stg[W2_TILE + w2_swz(e0 + j)] = a1[j]; }
            __syncthreads();
            uint32_t* d32 = reinterpret_cast<uint32_t*>(dlo + (O >= 4 ? per_op : 0)) + (O & 3);
            for (uint32_t e = t; e < W2_TILE; e += W2_THREADS) {
                const uint32_t q = w2_swz(e);
                *reinterpret_cast<uint2*>(d32 + 4 * e) = make_uint2(Stg[q], Stg[W2_TILE + q]);
            }
        }
    }
}

// changeRepr^-1 + InterleavedCombine: planes W (lo at W + p N, hi at + batch N) -> out (n_out = 2N words
// per product): out block w = lo128(C_w) ^ hi128(C_(w-1)), word 2w = limbs 0,1, word 2w+1 = limbs 2,3.
// Pairs run (4,5), (0,1), (6,7), (2,3): the hi pair of every element is staged before the lo pair that
// needs its predecessor's.  The tile's first element takes its predecessor from Hp (thread 0, tables).
// 4 thread groups of W2_THREADS share one tile: group g makes output limb pair O = {4, 6, 0, 2}[g] of its 32-element
// columns (the tile's planes are read by all four), so a CTA keeps 8 warps busy on 96 KB of shared memory
// (the one-group form held 2 warps per CTA on 80 KB).  The hi pairs (4,5), (6,7) are staged in H for the
// successor's lo pairs; the output words are staged limb-planar (in the plane area, free by then) and
// written coalesced.
#define IB2_GROUPS 4
#define IB2_THREADS (IB2_GROUPS * W2_THREADS)
#define IB2_SMEM (12 * W2_TILE * 4)
// MC (R28 on 128-bit blocks): out block j = lo128(C_j) ^ (M hi128(C))[j] in the novel basis,
// (M h)[j] = h[j-1] ^ [j odd] h[j] ^ [j even, j > 0] h[j + 2^ctz(j) - 1], for the 128-bit iBasisCvt that follows
template <bool MC>
__global__ void __launch_bounds__(IB2_THREADS, 1) k_ipsi256_bs(const uint4* __restrict__ W, uint64_t N, uint64_t batch,
                                                             const DevTables256* __restrict__ T, uint64_t* __restrict__ out) {
    extern __shared__ __align__(1024) uint32_t w2_smem[];
    uint32_t* In = w2_smem;                  // [8][W2_TILE] limb planes; afterwards [4][W2_TILE] output halves
    uint32_t* H = w2_smem + 8 * W2_TILE;     // [4][W2_TILE] hi pairs (4,5), (6,7) of every element
    __shared__ uint4 Hp;                     // predecessor's C hi128 (limbs 4..7)
    __shared__ uint4 Hf;                     // MC: the tile-aligned first block's far partner's hi128
    const uint64_t plane = batch * N, ntiles = plane / W2_TILE;
    const uint32_t t = threadIdx.x, g = t / W2_THREADS, e0 = 32 * (t % W2_THREADS);
    const int O = g == 0 ? 4 : (g == 1 ? 6 : (g == 2 ? 0 : 2));
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t g0 = tile * W2_TILE, p = g0 / N, i0 = g0 - p * N;
        const uint4* lo = W + g0;
        const uint4* hi = lo + plane;
        __syncthreads();   // the previous tile's output staging has been written out
        for (uint32_t e = t; e < W2_TILE; e += IB2_THREADS) {
            const uint4 a = lo[e], b = hi[e];
            const uint32_t q = w2_swz(e);
            In[q] = a.x; In[W2_TILE + q] = a.y; In[2 * W2_TILE + q] = a.z; In[3 * W2_TILE + q] = a.w;
            In[4 * W2_TILE + q] = b.x; In[5 * W2_TILE + q] = b.y; In[6 * W2_TILE + q] = b.z; In[7 * W2_TILE + q] = b.w;
        }
        if (t == 0) {
            uint4 rlo = make_uint4(0, 0, 0, 0), rhi = rlo;
            if (i0 != 0) ipsi256_apply(T->ipsi, lo[-1], hi[-1], rlo, rhi);   // (L1-cached global tables)
            Hp = rhi;
            uint4 flo = make_uint4(0, 0, 0, 0), fhi = flo;
            if (MC && i0 != 0) {
                const uint64_t d = (1ull << __ffsll((long long)i0) >> 1) - 1;   // 2^ctz(i0) - 1
                ipsi256_apply(T->ipsi, lo[d], hi[d], flo, fhi);
            }
            Hf = fhi;
        }
        __syncthreads();
        // limbs 2g, 2g + 1 of my column: elements -> planes, in place
#pragma unroll 1
        for (int L = 2 * (int)g; L < 2 * (int)g + 2; L++) {
            uint32_t x[32];
            w2_load_planes(In, L, e0, x);
            transpose32(x);
#pragma unroll
            for (int j = 0; j < 32; j++) In[L * W2_TILE + w2_swz(e0 + j)] = x[j];
        }
        __syncthreads();
        uint32_t a0[32], a1[32];
#pragma unroll
        for (int j = 0; j < 32; j++) { a0[j] = 0; a1[j] = 0; }
#pragma unroll 1
        for (int L = 0; L < 8; L++) {
            uint32_t x[32];
            w2_load_planes(In, L, e0, x);
            ipsi256_block(O, L, x, a0, a1);
        }
        transpose32(a0);
        transpose32(a1);
        if (O >= 4) {   // hi pair -> H[(O - 4) .. (O - 3)]
            uint32_t* h = H + (O - 4) * W2_TILE;
#pragma unroll
            for (int j = 0; j < 32; j++) { h[w2_swz(e0 + j)] = a0[j]; h[W2_TILE + w2_swz(e0 + j)] = a1[j]; }
        }
        __syncthreads();   // H complete; the planes are no longer read
        if (O < 4) {    // word 2e (O = 0: limbs 0,1 ^ C_(e-1) limbs 4,5) or 2e + 1 (O = 2: limbs 2,3 ^ limbs 6,7)
            const uint32_t* h = H + O * W2_TILE;
            const uint32_t* hp = reinterpret_cast<const uint32_t*>(&Hp) + O;
            const uint32_t* hf = reinterpret_cast<const uint32_t*>(&Hf) + O;
            uint32_t* o = In + O * W2_TILE;
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const uint32_t e = e0 + j;
                uint32_t p0 = e ? h[w2_swz(e - 1)] : hp[0];
                uint32_t p1 = e ? h[W2_TILE + w2_swz(e - 1)] : hp[1];
                if (MC && (i0 | e) != 0) {   // (tiles never straddle products: j = i0 + e)
                    if (e & 1) { p0 ^= h[w2_swz(e)]; p1 ^= h[W2_TILE + w2_swz(e)]; }
                    else if (e == 0) { p0 ^= hf[0]; p1 ^= hf[1]; }
                    else {
                        const uint32_t q = w2_swz(e + (e & (0u - e)) - 1);
                        p0 ^= h[q]; p1 ^= h[W2_TILE + q];
                    }
                }
                o[w2_swz(e)] = a0[j] ^ p0;
                o[W2_TILE + w2_swz(e)] = a1[j] ^ p1;
            }
        }
        __syncthreads();
        uint64_t* dst = out + p * 2 * N + 2 * i0;
        for (uint32_t i = t; i < 2 * W2_TILE; i += IB2_THREADS) {
            const uint32_t e = i >> 1, sel = (i & 1) * 2;
            dst[i] = ((uint64_t)In[(sel + 1) * W2_TILE + w2_swz(e)] << 32) | In[sel * W2_TILE + w2_swz(e)];
        }
    }
}

// ------------------------------------------------------------------------------ host pipeline
struct PlanW128 {
    uint64_t na, nb, ka, kb, N, batch;   // 64-bit words, 128-bit blocks per operand
    int m, ma, mb;
    std::vector<CvtPass> cvt_a, cvt_b, icvt;
    std::vector<FftPass> fft;
    size_t off_sa, off_sb, off_wa, off_wb, off_ta, off_tb, bytes;
};

static gf2x_status make_plan_w128(uint64_t a_bits, uint64_t b_bits, int64_t batch, PlanW128& P) {
    P.na = (a_bits + 63) / 64;
    P.nb = (b_bits + 63) / 64;
    P.ka = (a_bits + 127) / 128;
    P.kb = (b_bits + 127) / 128;
    P.batch = (uint64_t)batch;
    P.m = ceil_log2_u64(P.ka + P.kb - 1);
    if (P.m > 32) return fail(GF2X_ETOOBIG, "FFT size exceeds 2^32 points");
    P.N = 1ull << P.m;
    P.ma = ceil_log2_u64(P.ka);
    P.mb = ceil_log2_u64(P.kb);
    P.cvt_a = plan_cvt(P.ma, 16);
    P.cvt_b = plan_cvt(P.mb, 16);
    P.icvt = plan_cvt(P.m, 16);
    P.fft = plan_fft(P.m);
    const uint64_t B = P.batch;
    P.off_sa = 0;
    P.off_sb = P.off_sa + (1ull << P.ma) * B * 16;             // Sb directly after Sa
    P.off_wa = align256(P.off_sb + (1ull << P.mb) * B * 16);
    P.off_wb = P.off_wa + 2 * P.N * B * 16;                    // Wb directly after Wa
    P.off_ta = align256(P.off_wb + (2 * P.N * B + 2048) * 16);
    P.off_tb = P.off_ta + P.N * B * 16;                        // Tb directly after Ta
    P.bytes = align256(P.off_tb + (P.N * B + 2048) * 16);
    return GF2X_OK;
}

static gf2x_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GF2X_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return GF2X_OK;
}

static gf2x_status get_tables256(DeviceState* ds, DevTables256** out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!ds->tabs256) {
        DevTables256* h = new DevTables256;
        host_build_tables256(h);
        DevTables256* d = nullptr;
        cudaError_t e = cudaMalloc(&d, sizeof(DevTables256));
        if (e != cudaSuccess) { delete h; return fail(GF2X_ENOMEM, "table allocation failed"); }
        e = cudaMemcpy(d, h, sizeof(DevTables256), cudaMemcpyHostToDevice);
        delete h;
        if (e != cudaSuccess) { cudaFree(d); return fail(GF2X_ECUDA, cudaGetErrorString(e)); }
        CUDA_TRY(cudaFuncSetAttribute(k_w128_post, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_ipsi256_bs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, IB2_SMEM));
        CUDA_TRY(cudaFuncSetAttribute(k_ipsi256_bs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, IB2_SMEM));
        ds->tabs256 = d;
    }
    *out = ds->tabs256;
    return GF2X_OK;
}

static void bottom_run(uint4* A, uint4* B, uint64_t total, int m, int L, int mode, int smc, cudaStream_t st) {
    BottomParams bp;
    bp.A = A; bp.B = B;
    bp.total = total;
    bp.ntiles = (total + (1ull << BT_BITS) - 1) >> BT_BITS;
    bp.m = m; bp.L = L;
    bp.map = IdxMap{0, 0, 0};
    bp.mode = mode;
    const double bytes = (double)total * 16 * (((mode & 1) ? 4.0 : 0.0) + ((mode & 2) ? 3.0 : 0.0) + ((mode & 4) ? 2.0 : 0.0));
    ProfScope ps("k_bottom", bytes, st, bottom_alu_ops(bp));
    bottom_launch(bp, smc, st);
}

// stop_stage: 0 = product; 1 = after changeRepr, 2 = after FFT_LCH, 3 = after pointmul, 5 = after
// iBasisCvt (operand a's planes left in Wa)
// R28 for w = 128: the product fills all N blocks, whole bit-sliced tiles, a 16-byte aligned output
static bool w128_mcomb(const PlanW128& P, const uint64_t* c, int stop_stage) {
    return stop_stage == 0 && P.N % W2_TILE == 0 && P.na + P.nb == 2 * P.N && ((uintptr_t)c & 15) == 0 &&
           !env_flag("GF2X_NO_W2_BS") && !env_flag("GF2X_NO_MCOMB");
}
static gf2x_status run_pipeline_w128(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                     const PlanW128& P, void* ws, DeviceState* ds, cudaStream_t st, int stop_stage) {
    DevTables256* T256;
    gf2x_status s = get_tables256(ds, &T256);
    if (s != GF2X_OK) return s;
    unsigned char* base = reinterpret_cast<unsigned char*>(ws);
    uint4* Sa = reinterpret_cast<uint4*>(base + P.off_sa);
    uint4* Sb = reinterpret_cast<uint4*>(base + P.off_sb);
    uint4* Wa = reinterpret_cast<uint4*>(base + P.off_wa);
    uint4* Wb = reinterpret_cast<uint4*>(base + P.off_wb);
    uint4* Ta = reinterpret_cast<uint4*>(base + P.off_ta);
    uint4* Tb = reinterpret_cast<uint4*>(base + P.off_tb);
    const int smc = ds->sm_count;
    const uint64_t B = P.batch, plane = P.N * B;
    // Split into 128-bit blocks: the words, masked, zero-padded to 2^ma blocks
    {
        ProfScope ps("k_prep", (double)B * (P.na + (2ull << P.ma)) * 8, st);
        k_prep<<<grid_for((2ull << P.ma) * B, 256, smc, 8), 256, 0, st>>>(a, P.na, a_bits, P.ma + 1, B,
                                                                           reinterpret_cast<uint64_t*>(Sa));
    }
    {
        ProfScope ps("k_prep", (double)B * (P.nb + (2ull << P.mb)) * 8, st);
        k_prep<<<grid_for((2ull << P.mb) * B, 256, smc, 8), 256, 0, st>>>(b, P.nb, b_bits, P.mb + 1, B,
                                                                           reinterpret_cast<uint64_t*>(Sb));
    }
    if ((s = check_launch("prep")) != GF2X_OK) return s;
    // BasisCvt on the 128-bit blocks (XOR-only)
    const bool same = P.ma == P.mb;
    if (same) {
        if ((s = run_cvt<uint4>(P.cvt_a, Sa, P.ma, 2 * B, false, smc, st)) != GF2X_OK) return s;
    } else {
        if ((s = run_cvt<uint4>(P.cvt_a, Sa, P.ma, B, false, smc, st)) != GF2X_OK) return s;
        if ((s = run_cvt<uint4>(P.cvt_b, Sb, P.mb, B, false, smc, st)) != GF2X_OK) return s;
    }
    // changeRepr into TGF(2^256): bit-sliced when the tiles fit the products, else M4R-4
    const bool w2bs = P.N % W2_TILE == 0 && !env_flag("GF2X_NO_W2_BS");
    if (w2bs) {
        ProfScope ps("k_psi256_bs", (double)B * (((1ull << P.ma) + (1ull << P.mb)) * 16 + 2 * P.N * 32), st, 0.0, same ? 1 : 2);
        const size_t sm = 6 * W2_TILE * 4;
        if (same) {
            k_psi256_bs<<<grid_for(2 * plane / W2_TILE, 1, smc, 4), W2_THREADS, sm, st>>>(Sa, 1ull << P.ma, P.N, B, 2, Wa);
        } else {
            k_psi256_bs<<<grid_for(plane / W2_TILE, 1, smc, 4), W2_THREADS, sm, st>>>(Sa, 1ull << P.ma, P.N, B, 1, Wa);
            k_psi256_bs<<<grid_for(plane / W2_TILE, 1, smc, 4), W2_THREADS, sm, st>>>(Sb, 1ull << P.mb, P.N, B, 1, Wb);
        }
    } else if (same) {
        ProfScope ps("k_psi256", 2.0 * B * ((1ull << P.ma) * 16 + P.N * 32), st);
        k_psi256<<<grid_for(2 * plane, PSI256_THREADS, smc, 4), PSI256_THREADS, 0, st>>>(Sa, 1ull << P.ma, P.N, B, 2, T256, Wa);
    } else {
        ProfScope ps("k_psi256", (double)B * (((1ull << P.ma) + (1ull << P.mb)) * 16 + 2 * P.N * 32), st, 0.0, 2);
        k_psi256<<<grid_for(plane, PSI256_THREADS, smc, 4), PSI256_THREADS, 0, st>>>(Sa, 1ull << P.ma, P.N, B, 1, T256, Wa);
        k_psi256<<<grid_for(plane, PSI256_THREADS, smc, 4), PSI256_THREADS, 0, st>>>(Sb, 1ull << P.mb, P.N, B, 1, T256, Wb);
    }
    if ((s = check_launch("psi256")) != GF2X_OK) return s;
    if (stop_stage == 1) return GF2X_OK;
    // FFT_LCH top layers on the four plane sets (a lo/hi, b lo/hi) in one launch per pass
    Plan Pf;
    Pf.N = P.N; Pf.m = P.m; Pf.batch = 2 * B;
    const size_t ndirect = P.fft.size() - 1;
    for (size_t i = 0; i < ndirect; i++)
        if ((s = launch_fft(P.fft[i], false, false, Wa, P.N, Wa, Pf, ds, st, 2)) != GF2X_OK) return s;
    const int L = P.fft.back().layers;
    bottom_run(Wa, Wb, 2 * plane, P.m, L, 1, smc, st);
    if ((s = check_launch("bottom fwd")) != GF2X_OK) return s;
    if (stop_stage == 2) return GF2X_OK;
    // pointmul in TGF(2^256): Karatsuba over TGF(2^128)
    {
        ProfScope ps("k_w128_sums", 2.0 * plane * 48, st, 0.0, 2);
        k_w128_sums<<<grid_for(plane, 256, smc, 8), 256, 0, st>>>(Wa, plane, Ta);
        k_w128_sums<<<grid_for(plane, 256, smc, 8), 256, 0, st>>>(Wb, plane, Tb);
    }
    bottom_run(Wa, Wb, plane, P.m, L, 2, smc, st);                   // P0 = a_lo b_lo
    bottom_run(Wa + plane, Wb + plane, plane, P.m, L, 2, smc, st);   // P2 = a_hi b_hi
    bottom_run(Ta, Tb, plane, P.m, L, 2, smc, st);                   // P1
    {
        ProfScope ps("k_w128_post", (double)plane * 80, st);
        k_w128_post<<<grid_for(plane, 256, smc, 3), 256, 64 * 1024, st>>>(Wa, plane, Ta, T256);
    }
    if ((s = check_launch("pointmul256")) != GF2X_OK) return s;
    if (stop_stage == 3) return GF2X_OK;
    // iFFT_LCH: bottom layers, then the direct passes in reverse order
    bottom_run(Wa, Wa, 2 * plane, P.m, L, 4, smc, st);
    for (size_t i = ndirect; i-- > 0;)
        if ((s = launch_fft(P.fft[i], true, false, Wa, P.N, Wa, Pf, ds, st)) != GF2X_OK) return s;
    // R28: the combine in the novel basis into the output, then iBasisCvt of those 128-bit blocks in place (one plane
    // instead of two)
    if (w128_mcomb(P, c, stop_stage)) {
        {
            ProfScope ps("k_ipsi256_mcomb", 32.0 * plane + 16.0 * plane, st);
            k_ipsi256_bs<true><<<grid_for(plane / W2_TILE, 1, smc, 2), IB2_THREADS, IB2_SMEM, st>>>(Wa, P.N, B, T256, c);
        }
        if ((s = check_launch("ipsi256 mcomb")) != GF2X_OK) return s;
        return run_cvt<uint4>(P.icvt, reinterpret_cast<uint4*>(c), P.m, B, true, smc, st);
    }
    // iBasisCvt on both planes
    if ((s = run_cvt<uint4>(P.icvt, Wa, P.m, 2 * B, true, smc, st)) != GF2X_OK) return s;
    if (stop_stage == 5) return GF2X_OK;
    // changeRepr^-1 + InterleavedCombine
    if (w2bs && P.na + P.nb == 2 * P.N) {
        ProfScope ps("k_ipsi256_bs", 32.0 * plane + 16.0 * plane, st);
        k_ipsi256_bs<false><<<grid_for(plane / W2_TILE, 1, smc, 2), IB2_THREADS, IB2_SMEM, st>>>(Wa, P.N, B, T256, c);
    } else {
        const uint64_t n_out = P.na + P.nb, nblk = (n_out + 1) / 2;
        const uint64_t ctas = (nblk + IPSI256_THREADS - 1) / IPSI256_THREADS * B;
        ProfScope ps("k_ipsi256", 32.0 * plane + 8.0 * n_out * B, st);
        k_ipsi256<<<grid_for(ctas, 1, smc, 4), IPSI256_THREADS, 64 * 16 * 2 * 16, st>>>(Wa, P.N, B, n_out, T256, c);
    }
    return check_launch("ipsi256");
}

static gf2x_status mul_common_w128(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                   int64_t batch, void* stream, int stop_stage, uint64_t* stage_out) {
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
        if (out_bytes && !stop_stage) CUDA_TRY(cudaMemsetAsync(c, 0, out_bytes, st));
        return GF2X_OK;
    }
    int dev;
    DeviceState* ds;
    gf2x_status s = get_device(&dev, &ds);
    if (s != GF2X_OK) return s;
    PlanW128 P;
    if ((s = make_plan_w128(a_bits, b_bits, batch, P)) != GF2X_OK) return s;
    void* ws;
    if ((s = stream_workspace(ds, st, P.bytes, &ws)) != GF2X_OK) return s;
    if ((s = run_pipeline_w128(a, a_bits, b, b_bits, c, P, ws, ds, st, stop_stage)) != GF2X_OK) return s;
    if (stop_stage && stage_out) {   // (N, 4) words: element i = (lo plane i, hi plane i) of operand a, product 0
        const unsigned char* W = reinterpret_cast<unsigned char*>(ws) + P.off_wa;
        CUDA_TRY(cudaMemcpy2DAsync(stage_out, 32, W, 16, 16, P.N, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemcpy2DAsync(reinterpret_cast<unsigned char*>(stage_out) + 16, 32, W + P.N * P.batch * 16, 16, 16,
                                   P.N, cudaMemcpyDeviceToDevice, st));
    }
    return GF2X_OK;
}

static int launches_of_w128(const PlanW128& P) {
    const bool same = P.ma == P.mb;
    int n = 2;                                                     // prep
    n += cvt_launches(P.cvt_a, P.ma) + (same ? 0 : cvt_launches(P.cvt_b, P.mb));  // BasisCvt
    n += same ? 1 : 2;                                             // psi256
    const int nd = (int)P.fft.size() - 1;
    n += nd;                                                       // forward passes
    n += 1 + 2 + 3 + 1 + 1;                                        // bottom fwd, sums, 3 products, post, bottom inv
    n += nd + cvt_launches(P.icvt, P.m) + 1;                       // inverse passes, iBasisCvt, ipsi256
    return n;
}
