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
    // segmented conversions (CL >= 8; sm_conv_op): per op list (a, b, inverse) the mode (0: every op on the
    // whole array, 1: split, 2: the list lies inside segment 0) and the lengths of its top run and low block
    int cmode[3], ntop[3], nlow[3];
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
    L.pr = L.pl + 2 * 4 * GC * 33;       // the nine products: [GC][9][33]
    L.kd = L.pr + GC * 9 * 33;           // FFT constant deltas KD[layer < 9][2][16]
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
__device__ __forceinline__ void sm_consts(uint32_t c, uint32_t* K) {
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
// 2^K window identically, so the two commute (Kronecker factors).  With point segments of 2^mloc >= 2^K units
// each CTA runs the top run and the high block on the whole array (few ops) and the low block (most ops) on its
// own segment only; the inverse runs the inverted low block on its segment first, then the rest on the whole
// (gathered) array.  Step s of the forward schedule -> op index, and whether it runs segment-locally.
__device__ __forceinline__ int sm_conv_op(int s, int mode, int ntop, int nlow, int nops, bool& local) {
    local = mode == 2;
    if (mode != 1) return s;
    const int nhigh = nops - ntop - nlow;
    if (s < ntop) return s;
    if (s < ntop + nhigh) return ntop + nlow + (s - ntop);
    local = true;
    return ntop + (s - ntop - nhigh);
}

// Alg. 2 step (lg, K) on units of type T in s[0, 2^mm) as two sweeps, A (targets [h, h+u)) and B ([u, h)),
// source = target + d; forward A then B, inverse B then A (R4 / R7)
template <typename T>
__device__ __forceinline__ void sm_sweep(T* s, int mm, int lg, int K, bool A, int tid, int nthr) {
    const uint32_t h = 1u << (lg - 1), u = h >> K, d = h - u;
    const uint32_t nseg = 1u << (mm - lg);
    if (A) {
        const uint32_t n = nseg * u, lu = lg - 1 - K;   // u = 2^lu
        for (uint32_t it = tid; it < n; it += nthr) {
            const uint32_t seg = it >> lu, j = it & (u - 1);
            const uint32_t t = (seg << lg) + h + j;
            s[t] ^= s[t + d];
        }
    } else {
        const uint32_t n = nseg * h;
        for (uint32_t it = tid; it < n; it += nthr) {
            const uint32_t seg = it >> (lg - 1), j = it & (h - 1);
            if (j < u) continue;
            const uint32_t t = (seg << lg) + j;
            s[t] ^= s[t + d];
        }
    }
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
                                         const uint32_t* KD, uint32_t seg, uint32_t base, const uint32_t* KTk) {
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
                uint32_t x0 = x[i0], x1 = x[i1];
                if (INV) x1 ^= x0;
                x0 ^= sm_smul<W>(x1, K);
                if (!INV) x1 ^= x0;
                x[i0] = x0;
                x[i1] = x1;
            }
        }
    }
}
// layers [0, mloc) on the segment [base, base + 2^mloc) (mloc = m, base = 0: the whole transform)
template <bool INV>
__device__ __forceinline__ void sm_fft(uint32_t* A, uint32_t* B, int nops, int m, int LPC, uint32_t N, const uint32_t* KD,
                                       int mloc, uint32_t base, const uint32_t* KT) {
    const uint32_t seg = 1u << mloc;
    // layer k's KT entries start at kt_off(k): walked incrementally (up for the inverse, down for the forward)
    uint32_t kto = INV ? 0u : kt_off(m, mloc, mloc - 1);
    for (int s = 0; s < mloc; s++) {
        const int k = INV ? s : mloc - 1 - s;
        const int w = m - k;   // the layer's multipliers are < 2^w
        const uint32_t* KTk = KT ? KT + kto : nullptr;
        if (INV) kto += (seg >> (k + 1)) * (uint32_t)sm_width(w);
        else if (k > 0) kto -= (seg >> k) * (uint32_t)sm_width(w + 1);
        if (w <= 2) sm_layer<2, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk);
        else if (w <= 4) sm_layer<4, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk);
        else if (w <= 8) sm_layer<8, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk);
        else sm_layer<16, INV>(A, B, nops, m, k, LPC, N, KD, seg, base, KTk);
        __syncthreads();
    }
}

// The top log2 QC layers across the QC = CL / 4 segments of a limb (CL >= 8), y_s = value of segment s at a
// common offset.  Layer m-1 has the one block base 0 (multiplier 0: x1 ^= x0); layer m-2 has bases 0
// (multiplier 0) and 2^(m-1) (C = s_(m-2)(v_(m-1)), in GF(4)).  Forward (layers m-1, m-2, Alg. 1):
//   y0;  y1 ^ y0;  z2 = (y2 ^ y0) ^ C (y3 ^ y1);  (y3 ^ y1) ^ z2
// inverse (layers m-2, m-1):
//   y0;  y1 ^ y0;  (y2 ^ C (y3 ^ y2)) ^ y0;  (y3 ^ y2) ^ (y1 ^ y0)
// (QC = 2: layer m-1 only, y0; y1 ^ y0 both ways).  Every CTA reads the other segments' values over DSMEM
// into registers, the cluster barrier orders all reads before any write, then each writes its own segment.
#define SM_CROSS_MAXP 4
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
        for (int s = 0; s < QC; s++) src[s] = sm_limb<CL>(X, l0, s, N) + s * seg;
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
    sm_sync<CL>();   // every read of the old values done
    for (int o = 0; o < nops; o++) {
        uint32_t* X = (o ? B : A) + q * seg;
#pragma unroll
        for (int pi = 0; pi < SM_CROSS_MAXP; pi++) {
            const uint32_t i = threadIdx.x + pi * blockDim.x;
            if (i >= seg) break;
            X[i] = out[o][pi];
        }
    }
    __syncthreads();
}

template <int CL>
__global__ void __launch_bounds__(SM_THREADS, 1) k_small(SmallParams p) {
    extern __shared__ __align__(1024) uint32_t sm[];
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
    // ---- tables (once per CTA): psi (M4R-8: my limbs), psi^-1 (M4R-4, word-planar: entry (o, t, x) = limb o of
    // psi^-1(x << 4t) = limb o of the M4R-8 entry of byte t/2 with x in its nibble t&1)
    if (CL == 1) {
        for (int i = tid; i < 8 * 256; i += nthr) reinterpret_cast<uint4*>(ptab)[i] = p.tabs->psi64[i];
    } else {
        for (int i = tid; i < 8 * 256; i += nthr) ptab[i] = reinterpret_cast<const uint32_t*>(p.tabs->psi64 + i)[l0];
    }
    for (int i = tid; i < 4 * 32 * 16; i += nthr) {
        const int o = i >> 9, t = (i >> 4) & 31, x = i & 15;
        itab[i] = reinterpret_cast<const uint32_t*>(p.tabs->ipsi + (t >> 1) * 256 + (x << (4 * (t & 1))))[o];
    }
    if (tid < SM_KD_LAYERS * 2) {   // KD[k][i] = s_k(v_(9+i)) v_b, b < 16
        const int k = tid >> 1, i = tid & 1;
        uint32_t K[16];
        sm_consts<16>(k < 9 + i ? c_S[k * 32 + 9 + i] : 0u, K);
#pragma unroll
        for (int b = 0; b < 16; b++) KD[tid * 16 + b] = K[b];
    }
    if (KT) {   // the segment's FFT constants, once per CTA: layer k has 2^(mloc-k-1) blocks of sm_width(m-k) words
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
        // ---- 1 Split + pad
        const uint32_t ra = (uint32_t)(p.a_bits & 63), rb = (uint32_t)(p.b_bits & 63);
        for (uint32_t i = tid; i < N; i += nthr) {
            uint64_t x = i < p.na ? a[i] : 0ull, y = i < p.nb ? b[i] : 0ull;
            if (i == p.na - 1 && ra) x &= (1ull << ra) - 1;
            if (i == p.nb - 1 && rb) y &= (1ull << rb) - 1;
            SA[i] = x;
            SB[i] = y;
        }
        __syncthreads();
        // ---- 2 BasisCvt of both operands (every CTA of the cluster; with segments the low block on my segment only)
        for (int o = 0; o < max(p.nops_a, p.nops_b); o++)
            for (int ph = 0; ph < 2; ph++) {
#pragma unroll
                for (int x = 0; x < 2; x++) {
                    if (o >= (x ? p.nops_b : p.nops_a)) continue;
                    bool local;
                    const int oi = sm_conv_op(o, p.cmode[x], p.ntop[x], p.nlow[x], x ? p.nops_b : p.nops_a, local);
                    const CvtOp op = x ? p.ops_b[oi] : p.ops_a[oi];
                    uint64_t* S = x ? SB : SA;
                    const int mm = x ? p.mb : p.ma;
                    if (!local) sm_sweep<uint64_t>(S, mm, op.lg, op.K, ph == 0, tid, nthr);
                    else if (p.cmode[x] == 2) { if (q == 0) sm_sweep<uint64_t>(S, mm, op.lg, op.K, ph == 0, tid, nthr); }
                    else if ((sbase >> mm) == 0) sm_sweep<uint64_t>(S + sbase, m - QB, op.lg, op.K, ph == 0, tid, nthr);
                }
                __syncthreads();
            }
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
        // ---- 4 FFT_LCH of both spectra, my limbs (with segments: the top QB layers across them first)
        if constexpr (QB > 0) sm_cross<CL, false>(AL, BL, 2, m, q, l0, N);
        sm_fft<false>(AL, BL, 2, m, LPC, N, KD, m - QB, sbase, KT);
        sm_sync<CL>();   // every limb of A and B complete (pointmul reads them from every CTA)
        // ---- 5 pointmul, bit-sliced: my GC groups of 32 consecutive elements
        const uint32_t g0 = rank * GC;
        for (uint32_t it = tid; it < GC * 8; it += nthr) {   // (group, limb, operand): transpose into planes
            const uint32_t g = it >> 3, l = (it >> 1) & 3, o = it & 1;
            const uint32_t* src = sm_limb<CL>(o ? BL : AL, l, q, N) + ((g0 + g) << 5);
            uint32_t x[32];
#pragma unroll
            for (int j = 0; j < 32; j++) x[j] = src[j];
            transpose32(x);
            uint32_t* d = PL + ((o * 4 + l) * GC + g) * 33;
#pragma unroll
            for (int j = 0; j < 32; j++) d[j] = x[j];
        }
        __syncthreads();
        for (uint32_t it = tid; it < GC * 9; it += nthr) {   // (group, product): one bs_mul32 each
            const uint32_t g = it / 9, q = it - g * 9;
            const int mask = c_pm_terms[q][0];
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
            uint32_t* d = PR + (g * 9 + q) * 33;
#pragma unroll
            for (int j = 0; j < 32; j++) d[j] = r[j];
        }
        __syncthreads();
        for (uint32_t it = tid; it < GC * 4; it += nthr) {   // (group, result limb): R_L = sum of its terms
            const uint32_t g = it >> 2, L = it & 3;
            uint32_t acc[32], s1[32], s2[32], t[32];
#pragma unroll
            for (int j = 0; j < 32; j++) { acc[j] = 0; s1[j] = 0; s2[j] = 0; }
#pragma unroll 1
            for (int q = 0; q < 9; q++) {
                const uint32_t* src = PR + (g * 9 + q) * 33;
                const bool r0 = (c_pm_terms[q][1] >> L) & 1, r1 = (c_pm_terms[q][2] >> L) & 1, r2 = (c_pm_terms[q][3] >> L) & 1;
                if (r0) { for (int j = 0; j < 32; j++) acc[j] ^= src[j]; }
                if (r1) { for (int j = 0; j < 32; j++) s1[j] ^= src[j]; }
                if (r2) { for (int j = 0; j < 32; j++) s2[j] ^= src[j]; }
            }
            bs_mul_v31(s1, t);
#pragma unroll
            for (int j = 0; j < 32; j++) acc[j] ^= t[j];
            bs_mul_v31sq(s2, t);
#pragma unroll
            for (int j = 0; j < 32; j++) acc[j] ^= t[j];
            transpose32(acc);
            uint32_t* dst = sm_limb<CL>(AL, L, q, N) + ((g0 + g) << 5);
#pragma unroll
            for (int j = 0; j < 32; j++) dst[j] = acc[j];
        }
        sm_sync<CL>();   // every result limb delivered
        // ---- 6 iFFT_LCH, my limbs of the product (with segments: the top QB layers across them last, then
        // every CTA gathers its limb whole for iBasisCvt)
        sm_fft<true>(AL, BL, 1, m, LPC, N, KD, m - QB, sbase, KT);
        // ---- 7 iBasisCvt, my limbs (u32 units; XOR acts limb-wise); segmented (cmode[2] == 1): the inverted low
        // block on my segment, then the gather, then the inverted high block and top run on the whole limb
        int o_hi = p.nops_i - 1;
        if constexpr (QB > 0) {
            sm_cross<CL, true>(AL, BL, 1, m, q, l0, N);
            if (p.cmode[2] == 1) {
                const int lo = p.ntop[2], hi = p.ntop[2] + p.nlow[2];
                for (int o = hi - 1; o >= lo; o--)
                    for (int ph = 0; ph < 2; ph++) {
                        sm_sweep<uint32_t>(AL + sbase, m - QB, p.ops_i[o].lg, p.ops_i[o].K, ph == 1, tid, nthr);
                        __syncthreads();
                    }
            }
            sm_sync<CL>();   // every segment final
            for (uint32_t i = tid; i < N; i += nthr)
                if ((i >> (m - QB)) != q) AL[i] = sm_limb<CL>(AL, l0, i >> (m - QB), N)[i];
            __syncthreads();
        }
        for (int s = 0; s <= o_hi; s++) {
            int o = o_hi - s;   // reversed forward order; segmented: high block reversed, then top run reversed
            if (p.cmode[2] == 1) {
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
        sm_sync<CL>();   // (peers are done reading my limbs before they are overwritten / I exit)
    }
}
