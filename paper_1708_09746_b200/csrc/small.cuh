// small.cuh -- the whole Alg. 5 multiply of a product with N = 2^m <= 2^11 points in ONE kernel
// (SURVEY §7 step 3 / §3 call stack (4): "one fused kernel per product, the pipeline in shared memory"),
// included by gf2x.cu.
//
// A product runs on a cluster of CL CTAs (CL = 4 for a single product: CTA r owns limb r of both spectra;
// CL = 8 / 16: CTA r owns limb r % 4 of segment q = r / 4 of the points, QC = CL / 4 segments; CL = 1 for
// batches: one persistent CTA per product at a time, all four limbs).  Limbs are independent in every step
// except pointmul and changeRepr^-1 (Prop. 2: the FFT multipliers lie in TGF(2^32) and multiply each
// 32-bit limb on its own; BasisCvt is XOR only), so the cluster exchanges data twice, through distributed
// shared memory; with QC > 1 segments the top log2 QC FFT layers (block bases 0 and 2^(m-1): multipliers 0
// and s_(m-2)(v_(m-1)) in GF(4)) also cross segments, and iBasisCvt gathers each limb whole:
//   1 Split + pad          -> SA, SB (u64, zero-extended to N)
//   2 BasisCvt (Alg. 3 / Alg. 2)        -> in place on SA, SB (every CTA; Taylor steps as phase-A / phase-B sweeps)
//   3 changeRepr psi        -> my limbs of A, B (M4R-8 lookups of the product's psi tables)
//   4 FFT_LCH x2 (Alg. 1)     -> layers m-1 .. 0 on my limbs; multipliers s_k(phi(b)) < 2^(m-k) lie in
//                                          GF(2^16) (multiplier shortening P:802-815), multiplied by integer
//                                          products of the bits of each block (smul, fft.cuh)
//   5 pointmul              -> bit-sliced: 32 elements per plane word, the nine TGF(2^32) products of
//                                          the limb Karatsuba (bs_mul32) one per thread, combined per result limb
//   6 iFFT_LCH           -> layers 0 .. m-1 on my limbs of the product
//   7 iBasisCvt                 -> on my limbs (u32 units, reversed schedule, B then A)
//   8 changeRepr^-1 + combine -> every CTA a quarter of the output words (M4R-4, word-planar tables)
#pragma once

#define SM_THREADS 256
#define SM_MAX_OPS 48

struct SmallParams {
    const uint64_t* a;
    const uint64_t* b;
    uint64_t* c;
    uint64_t na, nb, a_bits, b_bits, batch;
    int m, ma, mb;
    int nops_a, nops_b, nops_i;
    int kt;   // 1: the FFT constants of the CTA's segment precomputed once into shared memory (KT)
    const uint32_t* ktg;   // (kt) the per-device copy of every segment's KT (get_small_kt): copied, not computed
    uint32_t ktw;          // its words per segment
    // split conversions (sm_conv_op): per op list (a, b, inverse) split[i] = 1: top run + high block
    // CTA-wide, low block (windows of 2^kw[i] units) warp by warp, on my segment only; 0: every op CTA-wide
    int split[3], ntop[3], nlow[3], kw[3];
    CvtOp ops_a[SM_MAX_OPS], ops_b[SM_MAX_OPS], ops_i[SM_MAX_OPS];
    const DevTables* tabs;
};

// width class of a layer's multipliers (< 2^w, w = m - k): the block width of the integer products
__host__ __device__ inline int sm_width(int w) { return w <= 2 ? 2 : (w <= 4 ? 4 : (w <= 8 ? 8 : 16)); }
// KT: for every local layer k < mloc and block of the segment (2^mloc points), the sm_width(m - k) constants
// K_b = c v_b of its multiplier c; layer k's entries start at kt_off(k) (32-bit words)
__host__ __device__ inline uint32_t kt_off(int m, int mloc, int k) {
    uint32_t o = 0;
    for (int j = 0; j < k; j++) o += (1u << (mloc - j - 1)) * (uint32_t)sm_width(m - j);
    return o;
}

// shared-memory layout (32-bit words), per CTA; N = 2^m, LPC = 4 / CL limbs (1 for CL >= 4), G = N / 32 groups,
// GC = G / CL
struct SmallLayout {
    uint32_t sa, sb, al, bl, ptab, itab, pl, pr, kd, kt, total;
};
__host__ __device__ inline int small_qb(int CL) { return CL == 16 ? 2 : (CL == 8 ? 1 : 0); }
__host__ __device__ inline SmallLayout small_layout(int m, int CL, bool kt = false) {
    SmallLayout L;
    const uint32_t N = 1u << m, LPC = CL >= 4 ? 1 : 4 / CL, GC = (N >> 5) / CL;
    L.sa = 0;
    L.sb = L.sa + 2 * N;
    L.al = L.sb + 2 * N;                 // [LPC][N]
    L.bl = L.al + LPC * N;
    L.ptab = L.bl + LPC * N;             // psi: CL = 1: uint4 M4R-8 (8 x 256 x 4 words); CL = 4: my limb (8 x 256)
    L.itab = L.ptab + (CL == 1 ? 8 * 256 * 4 : 8 * 256);   // psi^-1: M4R-4 word-planar [4 limbs][32 nibbles][16]
    L.pl = L.itab + 4 * 32 * 16;         // planes of A, B: [operand 2][limb 4][GC][33]
    L.pr = L.pl + 2 * 4 * GC * 33;       // the nine products P and v31 P, v31^2 P: [GC][9][3][33]
    L.kd = L.pr + GC * 27 * 33;          // FFT constant deltas KD[layer < 9][2][16]
    L.kt = (L.kd + 9 * 2 * 16 + 3) & ~3u;   // (kt) the segment's FFT constants (16-byte aligned)
    const int mloc = m - small_qb(CL);
    L.total = L.kt + (kt ? kt_off(m, mloc, mloc) : 0u);
    return L;
}

// ---- small-subfield constants: K_b = c v_b (tower basis v_b = prod of x_(i+1) over the bits i of b)
// SWAR products by the generators on 2-, 4-, 8- and 16-bit blocks (x_k^2 = x_k + x_1 ... x_(k-1))
// (mulx3 / mulx4 on bytes / 16-bit halves: gf2x_device.cuh)
// x0 ^= c x1 for a limb, c < 2^W: XOR over the bits b of every W-bit block of the integer products t_b K_b
template <int W>
__device__ __forceinline__ uint32_t sm_smul(uint32_t u, const uint32_t* K) {
    constexpr uint32_t M = W == 2 ? 0x55555555u : (W == 4 ? 0x11111111u : (W == 8 ? 0x01010101u : 0x00010001u));
    uint32_t r = (u & M) * K[0];
#pragma unroll
    for (int b = 1; b < W; b++) r ^= ((u >> b) & M) * K[b];
    return r;
}
template <int W>
__host__ __device__ __forceinline__ void sm_consts(uint32_t c, uint32_t* K) {
    K[0] = c;
    K[1] = mulx1(c);
    if constexpr (W > 2) {
        K[2] = mulx2(c);
        K[3] = mulx1(K[2]);
    }
    if constexpr (W > 4) {
#pragma unroll
        for (int b = 0; b < 4; b++) K[4 + b] = mulx3(K[b]);
    }
    if constexpr (W > 8) {
#pragma unroll
        for (int b = 0; b < 8; b++) K[8 + b] = mulx4(K[b]);
    }
}

template <int W>
__device__ __forceinline__ void sm_kt_store(uint32_t c, uint32_t* d) {
    uint32_t K[W];
    sm_consts<W>(c, K);
#pragma unroll
    for (int b = 0; b < W; b++) d[b] = K[b];
}

// BasisCvt's op list for 2^mm units (cvt_ops, gf2x.cu) is [top run: levels mm .. K+1 with K] [low block: the
// list for 2^K units, levels <= K] [high block: the list for the bits [K, mm), units of 2^K words].  The high
// block acts on the index bits >= K identically for every offset below 2^K, the low block inside every aligned
// 2^K window identically, so the two commute (Kronecker factors).  So the forward runs the top run and the
// high block CTA-wide (few ops, a barrier per sweep) and then the low block (most ops) window by window, one
// warp per window (__syncwarp between sweeps), only on the windows of my point segment; the inverse runs the
// inverted low block window by window first, then the rest CTA-wide on the whole (gathered) array.
// Step s of the CTA-wide forward schedule (split lists: top run, then high block) -> op index.
__device__ __forceinline__ int sm_conv_op(int s, int split, int ntop, int nlow) {
    return (!split || s < ntop) ? s : s + nlow;
}

// Alg. 2 step (lg, K) on units of type T in s[0, 2^mm) as two sweeps, A (targets [h, h+u)) and B ([u, h)),
// source = target + d; forward A then B, inverse B then A (R4 / R7)
template <typename T>
__device__ __forceinline__ void sm_sweep(T* s, int mm, int lg, int K, bool A, int tid, int nthr) {
    const uint32_t h = 1u << (lg - 1), u = h >> K, d = h - u;
    const uint32_t nseg = 1u << (mm - lg), lu = lg - 1 - K;   // u = 2^lu
    const uint32_t n = A ? nseg * u : nseg * h;
    // four targets per thread at a time: all loads first (a phase's targets and sources are disjoint and every
    // target is written once, so the loads of a batch may run ahead of its stores)
    for (uint32_t b0 = tid; b0 < n; b0 += 4 * nthr) {
        T v[4];
        uint32_t t[4];
        bool ok[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint32_t it = b0 + c * nthr;
            uint32_t seg, j;
            if (A) {
                seg = it >> lu; j = it & (u - 1);
                t[c] = (seg << lg) + h + j;
                ok[c] = it < n;
            } else {
                seg = it >> (lg - 1); j = it & (h - 1);
                t[c] = (seg << lg) + j;
                ok[c] = it < n && j >= u;
            }
            if (ok[c]) v[c] = s[t[c]] ^ s[t[c] + d];
        }
#pragma unroll
        for (int c = 0; c < 4; c++)
            if (ok[c]) s[t[c]] = v[c];
    }
}

// Alg. 2 step (LG, K) on 16 units held in registers (compile-time indices): sweeps A / B as sm_sweep
template <typename T, int LG, int K, bool A>
__device__ __forceinline__ void reg_sweep16(T* v) {
    constexpr int h = 1 << (LG - 1), u = h >> K, d = h - u, nseg = 1 << (4 - LG);
#pragma unroll
    for (int sg = 0; sg < nseg; sg++) {
        if (A) {
#pragma unroll
            for (int j = 0; j < u; j++) v[sg * 2 * h + h + j] ^= v[sg * 2 * h + h + j + d];
        } else {
#pragma unroll
            for (int j = u; j < h; j++) v[sg * 2 * h + j] ^= v[sg * 2 * h + j + d];
        }
    }
}
template <typename T, int LG, int K, bool INV>
__device__ __forceinline__ void reg_step16(T* v) {
    reg_sweep16<T, LG, K, !INV>(v);
    reg_sweep16<T, LG, K, INV>(v);
}
// BasisCvt of 16 units in registers: cvt_ops(4) = (4,2) (3,2) (2,1) (4,1); INV: its inverse
template <typename T, bool INV>
__device__ __forceinline__ void cvt16_regs(T* v) {
    if (!INV) {
        reg_step16<T, 4, 2, false>(v); reg_step16<T, 3, 2, false>(v); reg_step16<T, 2, 1, false>(v); reg_step16<T, 4, 1, false>(v);
    } else {
        reg_step16<T, 4, 1, true>(v); reg_step16<T, 2, 1, true>(v); reg_step16<T, 3, 2, true>(v); reg_step16<T, 4, 2, true>(v);
    }
}
// cvt16_regs on the 16 units w[off + i * str], i < 16
template <typename T, bool INV>
__device__ __forceinline__ void cvt16_pass(T* w, uint32_t off, uint32_t str) {
    T v[16];
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = w[off + i * str];
    cvt16_regs<T, INV>(v);
#pragma unroll
    for (int i = 0; i < 16; i++) w[off + i * str] = v[i];
}

// the low block (ops [ntop, ntop + nlow)) of a split list on the windows of 2^kw units in [lo, hi), a warp per
// window; INV: the inverted ops in reverse order.  Windows of 16 units (kw = 4: the block is cvt_ops(4)) run
// as one register pass per window; windows of 256 (kw = 8: cvt_ops(8) = [the 4 steps of levels 8..5]
// [cvt_ops(4) on bits 0..3][cvt_ops(4) on bits 4..7], the last two commuting Kronecker factors) as 4 swept
// steps and two register passes (16 units contiguous, then 16 units at stride 16)
template <typename T, bool INV>
__device__ __forceinline__ void sm_low_block(T* S, uint32_t lo, uint32_t hi, int kw, const CvtOp* ops, int ntop,
                                             int nlow, uint32_t nitems_before, uint32_t stride) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nwin = hi > lo ? (hi - lo) >> kw : 0;
    if (kw == 4) {   // a thread per 16-unit window (items counted in warps of 32 windows)
        const uint32_t nw32 = (nwin + 31) >> 5;
        for (uint32_t it = warp; it < nitems_before + nw32; it += stride) {
            if (it < nitems_before) continue;
            const uint32_t win = ((it - nitems_before) << 5) + lane;
            if (win < nwin) cvt16_pass<T, INV>(S + lo + (win << 4), 0, 1);
        }
        return;
    }
    for (uint32_t it = warp; it < nitems_before + nwin; it += stride) {
        if (it < nitems_before) continue;
        T* w = S + lo + ((it - nitems_before) << kw);
        const int nsw = kw == 8 ? 4 : nlow;   // swept steps (kw = 8: the top run of cvt_ops(8))
        if (kw == 8 && INV) {
            if (lane < 16) cvt16_pass<T, true>(w, lane, 16);
            __syncwarp();
            if (lane < 16) cvt16_pass<T, true>(w, lane << 4, 1);
            __syncwarp();
        }
        for (int j = 0; j < nsw; j++) {
            const CvtOp op = ops[ntop + (INV ? nsw - 1 - j : j)];
            sm_sweep<T>(w, kw, op.lg, op.K, !INV, lane, 32);
            __syncwarp();
            sm_sweep<T>(w, kw, op.lg, op.K, INV, lane, 32);
            __syncwarp();
        }
        if (kw == 8 && !INV) {
            if (lane < 16) cvt16_pass<T, false>(w, lane << 4, 1);
            __syncwarp();
            if (lane < 16) cvt16_pass<T, false>(w, lane, 16);
            __syncwarp();
        }
    }
}

// 32 x 32 bit transpose across a warp: lane j holds word j (row j) in, column j out (bit i = bit j of word i)
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int sh = 16; sh >= 1; sh >>= 1) {
        const uint32_t M = sh == 16 ? 0x0000FFFFu : (sh == 8 ? 0x00FF00FFu : (sh == 4 ? 0x0F0F0F0Fu : (sh == 2 ? 0x33333333u : 0x55555555u)));
        const uint32_t t = __shfl_xor_sync(0xffffffffu, v, sh);
        v = (lane & sh) ? ((v & ~M) | ((t & ~M) >> sh)) : ((v & M) | ((t & M) << sh));
    }
    return v;
}
__device__ __forceinline__ void sm_cp4(uint32_t* dst, const uint32_t* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <int CL>
__device__ __forceinline__ uint32_t* sm_peer(uint32_t* p, int rank) {
    if (CL == 1) return p;
    uint32_t* r;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
    return r;
}
// limb l of segment qq: its CTA's copy of the limb array X (CL >= 4: rank qq * 4 + l; CL = 1: limb l locally)
template <int CL>
__device__ __forceinline__ uint32_t* sm_limb(uint32_t* X, uint32_t l, uint32_t qq, uint32_t N) {
    if (CL == 1) return X + l * N;
    return sm_peer<CL>(X, qq * 4 + l);
}
template <int CL>
__device__ __forceinline__ void sm_sync() {
    if (CL == 1) __syncthreads();
    else asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// one FFT layer k on my limbs of A (and B): forward x0 ^= c x1, x1 ^= x0; inverse x1 ^= x0, x0 ^= c x1.
// Thread t takes the butterflies it = t + 256 j: their block bases are b_0 | j 2^9 (b_0 < 2^9), so by the
// linearity of s_k and of c -> c v_b the constants are K(j) = K(0) ^ [j & 1] KD[k][0] ^ [j & 2] KD[k][1] with
// KD[k][i][b] = s_k(v_(9+i)) v_b (layers k <= 8; built once per CTA): one full constant per thread and layer.
#define SM_KD_LAYERS 9
template <int W, bool INV>
__device__ __forceinline__ void sm_layer(uint32_t* A, uint32_t* B, int nops, int m, int k, int LPC, uint32_t N,
                                         const uint32_t* KD, uint32_t seg, uint32_t base, const uint32_t* KTk,
                                         int dsh) {
    const uint32_t half = seg >> 1;   // butterflies of the segment [base, base + seg)
    uint32_t K0[W];
    bool have = false;
    for (uint32_t it = threadIdx.x, j = 0; it < half; it += blockDim.x, j++) {
        const uint32_t blk = it >> k, off = it & ((1u << k) - 1);
        const uint32_t i0 = base + ((blk << (k + 1)) | off), i1 = i0 | (1u << k);
        uint32_t K[W];
        if (KTk) {   // precomputed (16-byte aligned entries for W >= 4)
            if constexpr (W == 2) {
                const uint2 v = reinterpret_cast<const uint2*>(KTk)[blk];
                K[0] = v.x;
                K[1] = v.y;
            } else {
#pragma unroll
                for (int b = 0; b < W; b += 4) {
                    const uint4 v = reinterpret_cast<const uint4*>(KTk + blk * W)[b >> 2];
                    K[b] = v.x; K[b + 1] = v.y; K[b + 2] = v.z; K[b + 3] = v.w;
                }
            }
        } else if (blockDim.x == 256 && k < SM_KD_LAYERS && have) {
#pragma unroll
            for (int b = 0; b < W; b++)
                K[b] = K0[b] ^ ((j & 1) ? KD[(k * 2 + 0) * 16 + b] : 0u) ^ ((j & 2) ? KD[(k * 2 + 1) * 16 + b] : 0u);
        } else {
            const uint32_t cst = layer_const(k, base + (blk << (k + 1)));
            sm_consts<W>(cst, K);
            if (j == 0) {
#pragma unroll
                for (int b = 0; b < W; b++) K0[b] = K[b];
                have = true;
            }
        }
        for (int o = 0; o < nops; o++) {
            uint32_t* X = o ? B : A;
            for (int l = 0; l < LPC; l++) {
                uint32_t* x = X + l * N;
                const uint32_t j0 = i0 + dsh, j1 = i1 + dsh;   // (data of the segment at base + dsh)
                uint32_t x0 = x[j0], x1 = x[j1];
                if (INV) x1 ^= x0;
                x0 ^= sm_smul<W>(x1, K);
                if (!INV) x1 ^= x0;
                x[j0] = x0;
                x[j1] = x1;
            }
        }
    }
}
// layers [0, mloc) on the segment [base, base + 2^mloc) (mloc = m, base = 0: the whole transform), its data
// stored at base + dsh (radix-4 layer pairs with one barrier each measured slower: 39.2 against 32.8 us at c1)
template <bool INV>
__device__ __forceinline__ void sm_fft(uint32_t* A, uint32_t* B, int nops, int m, int LPC, uint32_t N, const uint32_t* KD,
                                       int mloc, uint32_t base, const uint32_t* KT, int dsh) {
    const uint32_t seg = 1u << mloc;
    // layer k's KT entries start at kt_off(k): walked incrementally (up for the inverse, down for the forward)
    uint32_t kto = INV ? 0u : kt_off(m, mloc, mloc - 1);
    for (int s = 0; s < mloc; s++) {
        const int k = INV ? s : mloc - 1 - s;
        const int w = m - k;   // the layer's multipliers are < 2^w
        const uint32_t* KTk = KT ? KT + kto : nullptr;
        if (INV) kto += (seg >> (k + 1)) * (uint32_t)sm_width(w);
        else if (k > 0) kto -= (seg >> k) * (uint32_t)sm_width(w + 1);
        if (w <= 2) sm_layer<2, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk, dsh);
        else if (w <= 4) sm_layer<4, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk, dsh);
        else if (w <= 8) sm_layer<8, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk, dsh);
        else sm_layer<16, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk, dsh);
        __syncthreads();
    }
}

// The top log2 QC layers across the QC = CL / 4 segments of a limb (CL >= 8), y_s = value of segment s at a
// common offset.  Layer m-1 has the one block base 0 (multiplier 0: x1 ^= x0); layer m-2 has bases 0
// (multiplier 0) and 2^(m-1) (C = s_(m-2)(v_(m-1)), in GF(4)).  Forward (layers m-1, m-2, Alg. 1):
//   y0;  y1 ^ y0;  z2 = (y2 ^ y0) ^ C (y3 ^ y1);  (y3 ^ y1) ^ z2
// inverse (layers m-2, m-1):
//   y0;  y1 ^ y0;  (y2 ^ C (y3 ^ y2)) ^ y0;  (y3 ^ y2) ^ (y1 ^ y0)
// (QC = 2: layer m-1 only, y0; y1 ^ y0 both ways).  Every CTA reads the other segments' values over DSMEM.
// Double-buffered: segment s's canonical region is [s seg, (s+1) seg) of its limb arrays, its working region
// (where its FFT layers run, between the two cross steps) the region of segment (s+1) mod QC of the SAME
// arrays (free then: each CTA only holds its own segment).  The forward cross reads canonical regions and
// writes the working one, the inverse reads working regions and writes the canonical one, so no CTA ever
// writes a region a peer is reading and one cluster barrier (inputs complete) suffices.
#define SM_CROSS_MAXP 4
__host__ __device__ inline uint32_t sm_wreg(uint32_t s, int QC) { return (s + 1) & (uint32_t)(QC - 1); }
template <int CL, bool INV>
__device__ __forceinline__ void sm_cross(uint32_t* A, uint32_t* B, int nops, int m, uint32_t q, uint32_t l0,
                                         uint32_t N) {
    constexpr int QC = CL / 4;
    const uint32_t seg = N / QC;
    uint32_t K[2] = {0u, 0u};
    if (QC == 4) sm_consts<2>(layer_const(m - 2, 1u << (m - 1)), K);
    uint32_t out[2][SM_CROSS_MAXP];
    sm_sync<CL>();   // every segment's input complete
    for (int o = 0; o < nops; o++) {
        uint32_t* X = o ? B : A;
        const uint32_t* src[QC];
#pragma unroll
        for (int s = 0; s < QC; s++) src[s] = sm_limb<CL>(X, l0, s, N) + (INV ? sm_wreg(s, QC) : s) * seg;
#pragma unroll
        for (int pi = 0; pi < SM_CROSS_MAXP; pi++) {
            const uint32_t i = threadIdx.x + pi * blockDim.x;
            if (i >= seg) break;
            uint32_t y[QC];
#pragma unroll
            for (int s = 0; s < QC; s++) y[s] = src[s][i];
            uint32_t r = y[0];
            if constexpr (QC == 2) {
                if (q == 1) r = y[1] ^ y[0];
            } else if (!INV) {
                const uint32_t t2 = y[2] ^ y[0], t3 = y[3] ^ y[1];
                const uint32_t z2 = t2 ^ sm_smul<2>(t3, K);
                r = q == 0 ? y[0] : (q == 1 ? y[1] ^ y[0] : (q == 2 ? z2 : t3 ^ z2));
            } else {
                const uint32_t t3 = y[3] ^ y[2];
                r = q == 0 ? y[0] : (q == 1 ? y[1] ^ y[0] : (q == 2 ? (y[2] ^ sm_smul<2>(t3, K)) ^ y[0] : t3 ^ y[1] ^ y[0]));
            }
            out[o][pi] = r;
        }
    }
    for (int o = 0; o < nops; o++) {
        uint32_t* X = (o ? B : A) + (INV ? q : sm_wreg(q, QC)) * seg;
#pragma unroll
        for (int pi = 0; pi < SM_CROSS_MAXP; pi++) {
            const uint32_t i = threadIdx.x + pi * blockDim.x;
            if (i >= seg) break;
            X[i] = out[o][pi];
        }
    }
    __syncthreads();
}

// SM_TRACE builds (tools/dev/small_trace.py): %globaltimer of thread 0 of every CTA at the phase ends
#ifdef SM_TRACE
__device__ unsigned long long g_sm_trace[16][16];
#define SM_T(i)                                                                                              \
    do {                                                                                                     \
        if (threadIdx.x == 0 && blockIdx.x < 16) {                                                           \
            unsigned long long t_;                                                                           \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                           \
            g_sm_trace[blockIdx.x][i] = t_;                                                                  \
        }                                                                                                    \
    } while (0)
#else
#define SM_T(i) do {} while (0)
#endif
template <int CL>
__global__ void __launch_bounds__(SM_THREADS, 1) k_small(SmallParams p) {
    extern __shared__ __align__(1024) uint32_t sm[];
    SM_T(0);
    const int m = p.m;
    constexpr int QC = CL >= 8 ? CL / 4 : 1;   // segments of the points
    constexpr int QB = QC == 4 ? 2 : (QC == 2 ? 1 : 0);
    const uint32_t N = 1u << m, LPC = CL >= 4 ? 1 : 4 / CL, G = N >> 5, GC = G / CL;
    const SmallLayout Ly = small_layout(m, CL, p.kt != 0);
    uint64_t* SA = reinterpret_cast<uint64_t*>(sm + Ly.sa);
    uint64_t* SB = reinterpret_cast<uint64_t*>(sm + Ly.sb);
    uint32_t* AL = sm + Ly.al;
    uint32_t* BL = sm + Ly.bl;
    uint32_t* ptab = sm + Ly.ptab;
    uint32_t* itab = sm + Ly.itab;
    uint32_t* PL = sm + Ly.pl;
    uint32_t* PR = sm + Ly.pr;
    uint32_t* KD = sm + Ly.kd;
    uint32_t* KT = p.kt ? sm + Ly.kt : nullptr;
    uint32_t rank = 0;
    if (CL > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int tid = threadIdx.x, nthr = blockDim.x;
    const uint32_t l0 = CL >= 4 ? (rank & 3) : 0;   // my first limb
    const uint32_t q = CL >= 4 ? (rank >> 2) : 0;    // my segment of the points
    const uint32_t seg = N >> QB, sbase = q * seg;
    // with segments, the FFT data lives in the working region between the cross steps (sm_cross)
    const int dsh = QB ? (int)(sm_wreg(q, QC) * seg) - (int)sbase : 0;
    // ---- tables (once per CTA): psi (M4R-8: my limbs), psi^-1 (M4R-4, word-planar: entry (o, t, x) = limb o of
    // psi^-1(x << 4t) = limb o of the M4R-8 entry of byte t/2 with x in its nibble t&1)
    // (asynchronous copies: they complete under the constant builds, Split and BasisCvt; waited before psi)
    if (CL == 1) {
        for (int i = tid; i < 8 * 256; i += nthr) cp_async16(reinterpret_cast<uint4*>(ptab) + i, p.tabs->psi64 + i);
    } else {
        for (int i = tid; i < 8 * 256; i += nthr) sm_cp4(ptab + i, reinterpret_cast<const uint32_t*>(p.tabs->psi64 + i) + l0);
    }
    for (int i = tid; i < 4 * 32 * 16; i += nthr) {
        const int o = i >> 9, t = (i >> 4) & 31, x = i & 15;
        sm_cp4(itab + i, reinterpret_cast<const uint32_t*>(p.tabs->ipsi + (t >> 1) * 256 + (x << (4 * (t & 1)))) + o);
    }
    cp_async_commit();
    if (!KT && tid < SM_KD_LAYERS * 2) {   // KD[k][i] = s_k(v_(9+i)) v_b, b < 16 (without KT only)
        const int k = tid >> 1, i = tid & 1;
        uint32_t K[16];
        sm_consts<16>(k < 9 + i ? c_S[k * 32 + 9 + i] : 0u, K);
#pragma unroll
        for (int b = 0; b < 16; b++) KD[tid * 16 + b] = K[b];
    }
    if (KT && p.ktg) {   // the segment's FFT constants: copied from the per-device table (asynchronously)
        const uint4* src = reinterpret_cast<const uint4*>(p.ktg + (size_t)q * p.ktw);
        for (uint32_t i = tid; i < (p.ktw >> 2); i += nthr) cp_async16(reinterpret_cast<uint4*>(KT) + i, src + i);
        cp_async_commit();
    } else if (KT) {   // ... or built once per CTA: layer k has 2^(mloc-k-1) blocks of sm_width(m-k) words
        const int mloc = m - QB;
        for (uint32_t i = tid; i < seg - 1; i += nthr) {
            int k = 0;
            uint32_t blk = i;
            while (blk >= (seg >> (k + 1))) { blk -= seg >> (k + 1); k++; }
            const uint32_t cst = layer_const(k, sbase + (blk << (k + 1)));
            const int W = sm_width(m - k);
            uint32_t* d = KT + kt_off(m, mloc, k) + blk * W;
            if (W == 2) sm_kt_store<2>(cst, d);
            else if (W == 4) sm_kt_store<4>(cst, d);
            else if (W == 8) sm_kt_store<8>(cst, d);
            else sm_kt_store<16>(cst, d);
        }
    }
    const uint64_t n_out = p.na + p.nb;
    const uint64_t pstep = CL == 1 ? gridDim.x : gridDim.x / CL;
    for (uint64_t pr = CL == 1 ? blockIdx.x : blockIdx.x / CL; pr < p.batch; pr += pstep) {
        const uint64_t* a = p.a + pr * p.na;
        const uint64_t* b = p.b + pr * p.nb;
        __syncthreads();   // (tables; the previous product's last reads of SA .. PR)
        SM_T(1);
        // ---- 1 Split + pad (asynchronous copies; the last word of an operand with a partial top word masked)
        const uint32_t ra = (uint32_t)(p.a_bits & 63), rb = (uint32_t)(p.b_bits & 63);
        for (uint32_t i = tid; i < N; i += nthr) {
            if (i >= p.na) SA[i] = 0ull;
            else if (i == p.na - 1 && ra) SA[i] = a[i] & ((1ull << ra) - 1);
            else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(SA + i)), "l"(a + i) : "memory");
            if (i >= p.nb) SB[i] = 0ull;
            else if (i == p.nb - 1 && rb) SB[i] = b[i] & ((1ull << rb) - 1);
            else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(SB + i)), "l"(b + i) : "memory");
        }
        cp_async_commit();
        cp_async_wait<0>();   // (also the tables, on the first product)
        __syncthreads();
        SM_T(2);
        // ---- 2 BasisCvt of both operands (every CTA of the cluster; with segments the low block on my segment only)
        {
            // CTA-wide steps (a CTA whose segment lies past an operand skips it: its part stays zero)
            const int na_cta = p.split[0] ? p.nops_a - p.nlow[0] : p.nops_a;
            const int nb_cta = p.split[1] ? p.nops_b - p.nlow[1] : p.nops_b;
            for (int o = 0; o < max(na_cta, nb_cta); o++)
                for (int ph = 0; ph < 2; ph++) {
#pragma unroll
                    for (int x = 0; x < 2; x++) {
                        const int mm = x ? p.mb : p.ma;
                        if (o >= (x ? nb_cta : na_cta) || (sbase >> mm) != 0) continue;
                        const int oi = sm_conv_op(o, p.split[x], p.ntop[x], p.nlow[x]);
                        const CvtOp op = x ? p.ops_b[oi] : p.ops_a[oi];
                        sm_sweep<uint64_t>(x ? SB : SA, mm, op.lg, op.K, ph == 0, tid, nthr);
                    }
                    __syncthreads();
                }
            // the low blocks, window by window on my segment's part of each operand
            uint32_t before = 0;
#pragma unroll
            for (int x = 0; x < 2; x++) {
                if (!p.split[x]) continue;
                const uint32_t ext = 1u << (x ? p.mb : p.ma);
                const uint32_t lo = QB ? sbase : 0u, hi = min(lo + seg, ext);
                sm_low_block<uint64_t, false>(x ? SB : SA, lo, hi, p.kw[x], x ? p.ops_b : p.ops_a, p.ntop[x], p.nlow[x],
                                              before, nthr >> 5);
                const uint32_t nw = hi > lo ? (hi - lo) >> p.kw[x] : 0;
                before += p.kw[x] == 4 ? (nw + 31) >> 5 : nw;   // (sm_low_block's work items)
            }
            __syncthreads();
        }
            SM_T(3);
        // ---- 3 changeRepr: my limbs of psi(SA[i]), psi(SB[i]), i in my segment
        for (uint32_t i = sbase + tid; i < sbase + seg; i += nthr) {
            const uint64_t x = SA[i], y = SB[i];
            for (uint32_t l = 0; l < LPC; l++) {
                uint32_t va = 0, vb = 0;
#pragma unroll
                for (int ch = 0; ch < 8; ch++) {
                    const uint32_t ia = (uint32_t)(x >> (8 * ch)) & 255, ib = (uint32_t)(y >> (8 * ch)) & 255;
                    if (CL == 1) {
                        va ^= ptab[(ch * 256 + ia) * 4 + l];
                        vb ^= ptab[(ch * 256 + ib) * 4 + l];
                    } else {
                        va ^= ptab[ch * 256 + ia];
                        vb ^= ptab[ch * 256 + ib];
                    }
                }
                AL[l * N + i] = va;
                BL[l * N + i] = vb;
            }
        }
        __syncthreads();
        SM_T(4);
        // ---- 4 FFT_LCH of both spectra, my limbs (with segments: the top QB layers across them first)
        if constexpr (QB > 0) sm_cross<CL, false>(AL, BL, 2, m, q, l0, N);
        SM_T(5);
        sm_fft<false>(AL, BL, 2, m, LPC, N, KD, m - QB, sbase, KT, dsh);
        sm_sync<CL>();   // every limb of A and B complete (pointmul reads them from every CTA)
        SM_T(6);
        // ---- 5 pointmul, bit-sliced: my GC groups of 32 consecutive elements
        const uint32_t g0 = rank * GC;
        const uint32_t lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
        for (uint32_t it = warp; it < GC * 8; it += nwarp) {   // (group, limb, operand): a warp transposes into planes
            const uint32_t g = it >> 3, l = (it >> 1) & 3, o = it & 1;
            const uint32_t* src = sm_limb<CL>(o ? BL : AL, l, q, N) + (int)((g0 + g) << 5) + dsh;
            PL[((o * 4 + l) * GC + g) * 33 + lane] = warp_transpose32(src[lane], lane);
        }
        __syncthreads();
        SM_T(7);
        for (uint32_t it = tid; it < GC * 9; it += nthr) {   // (group, product): one bs_mul32 each
            const uint32_t g = it / 9, qq = it - g * 9;
            const int mask = c_pm_terms[qq][0];
            uint32_t x[32], y[32], r[32];
#pragma unroll
            for (int j = 0; j < 32; j++) { x[j] = 0; y[j] = 0; }
#pragma unroll
            for (int l = 0; l < 4; l++)
                if (mask & (1 << l)) {
                    const uint32_t* pa = PL + ((0 * 4 + l) * GC + g) * 33;
                    const uint32_t* pb = PL + ((1 * 4 + l) * GC + g) * 33;
#pragma unroll
                    for (int j = 0; j < 32; j++) { x[j] ^= pa[j]; y[j] ^= pb[j]; }
                }
            bs_mul32(x, y, r);
            uint32_t* d = PR + (g * 9 + qq) * 3 * 33;
#pragma unroll
            for (int j = 0; j < 32; j++) d[j] = r[j];
            // the product scaled by the Karatsuba constants where a result limb takes it so (combine below)
            if (c_pm_terms[qq][2]) {
                bs_mul_v31(r, x);
#pragma unroll
                for (int j = 0; j < 32; j++) d[33 + j] = x[j];
            }
            if (c_pm_terms[qq][3]) {
                bs_mul_v31sq(r, x);
#pragma unroll
                for (int j = 0; j < 32; j++) d[66 + j] = x[j];
            }
        }
        __syncthreads();
        SM_T(8);
        // (group, result limb): R_L = sum of its terms P, v31 P, v31^2 P (c_pm_terms), a warp per item with lane j
        // on plane j, then a warp transpose back to elements
        for (uint32_t it = warp; it < GC * 4; it += nwarp) {
            const uint32_t g = it >> 2, L = it & 3;
            uint32_t acc = 0;
#pragma unroll
            for (int t9 = 0; t9 < 9; t9++) {
                const uint32_t* src = PR + (g * 9 + t9) * 3 * 33 + lane;
                if ((c_pm_terms[t9][1] >> L) & 1) acc ^= src[0];
                if ((c_pm_terms[t9][2] >> L) & 1) acc ^= src[33];
                if ((c_pm_terms[t9][3] >> L) & 1) acc ^= src[66];
            }
            uint32_t* dst = sm_limb<CL>(AL, L, q, N) + (int)((g0 + g) << 5) + dsh;
            dst[lane] = warp_transpose32(acc, lane);
        }
        sm_sync<CL>();   // every result limb delivered
        SM_T(9);
        // ---- 6 iFFT_LCH, my limbs of the product (with segments: the top QB layers across them last, then
        // every CTA gathers its limb whole for iBasisCvt)
        sm_fft<true>(AL, BL, 1, m, LPC, N, KD, m - QB, sbase, KT, dsh);
        SM_T(10);
        // ---- 7 iBasisCvt, my limbs (u32 units; XOR acts limb-wise); segmented (cmode[2] == 1): the inverted low
        // block on my segment, then the gather, then the inverted high block and top run on the whole limb
        int o_hi = p.nops_i - 1;
        if constexpr (QB > 0) sm_cross<CL, true>(AL, BL, 1, m, q, l0, N);
        if (p.split[2]) {   // the inverted low block, window by window on my segment (every limb I hold)
            for (uint32_t l = 0; l < LPC; l++)
                sm_low_block<uint32_t, true>(AL + l * N, sbase, sbase + seg, p.kw[2], p.ops_i, p.ntop[2], p.nlow[2],
                                             l * (p.kw[2] == 4 ? ((seg >> 4) + 31) >> 5 : seg >> p.kw[2]), nthr >> 5);
            __syncthreads();
        }
        if constexpr (QB > 0) {
            sm_sync<CL>();   // every segment final
            SM_T(11);
            for (uint32_t i = tid; i < N; i += nthr)
                if ((i >> (m - QB)) != q) AL[i] = sm_limb<CL>(AL, l0, i >> (m - QB), N)[i];
            __syncthreads();
            SM_T(12);
        }
        for (int s = 0; s <= o_hi; s++) {
            int o = o_hi - s;   // reversed forward order; split: high block reversed, then top run reversed
            if (p.split[2]) {
                const int nhigh = p.nops_i - p.ntop[2] - p.nlow[2];
                if (s < nhigh) o = p.nops_i - 1 - s;
                else if (s < nhigh + p.ntop[2]) o = p.ntop[2] - 1 - (s - nhigh);
                else break;
            }
            for (int ph = 0; ph < 2; ph++) {
                for (uint32_t l = 0; l < LPC; l++)
                    sm_sweep<uint32_t>(AL + l * N, m, p.ops_i[o].lg, p.ops_i[o].K, ph == 1, tid, nthr);
                __syncthreads();
            }
        }
        sm_sync<CL>();   // every limb of the product converted
        SM_T(13);
        // ---- 8 changeRepr^-1 + InterleavedCombine: out[w] = lo64(C_w) ^ hi64(C_(w-1)), C_i = 0 for i >= N
        const uint32_t* Lp[4];
#pragma unroll
        for (int l = 0; l < 4; l++) Lp[l] = sm_limb<CL>(AL, l, q, N);
        uint64_t* cout = p.c + pr * n_out;
        const uint32_t wpc = (uint32_t)((n_out + CL - 1) / CL);
        for (uint32_t w = rank * wpc + tid; w < min((uint64_t)(rank + 1) * wpc, n_out); w += nthr) {
            uint32_t lo0 = 0, lo1 = 0, hi2 = 0, hi3 = 0;
            if (w < N) {
                uint32_t v[4];
#pragma unroll
                for (int l = 0; l < 4; l++) v[l] = Lp[l][w];
#pragma unroll
                for (int t = 0; t < 32; t++) {
                    const uint32_t x = (v[t >> 3] >> (4 * (t & 7))) & 15;
                    lo0 ^= itab[(0 * 32 + t) * 16 + x];
                    lo1 ^= itab[(1 * 32 + t) * 16 + x];
                }
            }
            if (w >= 1 && w - 1 < N) {
                uint32_t v[4];
#pragma unroll
                for (int l = 0; l < 4; l++) v[l] = Lp[l][w - 1];
#pragma unroll
                for (int t = 0; t < 32; t++) {
                    const uint32_t x = (v[t >> 3] >> (4 * (t & 7))) & 15;
                    hi2 ^= itab[(2 * 32 + t) * 16 + x];
                    hi3 ^= itab[(3 * 32 + t) * 16 + x];
                }
            }
            cout[w] = ((uint64_t)(lo1 ^ hi3) << 32) | (lo0 ^ hi2);
        }
        SM_T(14);
        sm_sync<CL>();   // (peers are done reading my limbs before they are overwritten / I exit)
        SM_T(15);
    }
}
