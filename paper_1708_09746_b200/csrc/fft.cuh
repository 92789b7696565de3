// fft.cuh -- FFT_LCH / iFFT_LCH passes (Alg. 1, inverse P:408), included by gf2x.cu.
//
// A pass handles the layers k_hi-1 .. k_lo of tiles with index bits [0,c) U [k_lo,k_hi) (c >= 5,
// k_lo >= the bottom layers) held in shared memory.  All lanes of a warp work on different columns (bits < c)
// of the same rows, so every multiplier is warp-uniform; the 2^R - 1 distinct multipliers of a tile
// (one per block per layer) get one M4R-4 table each, built once per tile.  The layers below
// that run in the fused bit-sliced bottom kernel (bottom.cuh).
// Inside a pass the layers run in groups of up to three: each thread holds the 2^r elements of a
// radix-2^r sub-transform in registers, so shared-memory traffic is one load/store per element per
// group instead of per layer.
//
// Butterfly (forward): x0 ^= c x1; x1 ^= x0   (second multiplier s_k(v_k) = 1, Prop. 1)
//           (inverse): x1 ^= x0; x0 ^= c x1
#pragma once

#define FFT_THREADS 256
#define FFT_UNR 8
#ifndef FFT_PSI_PF
#define FFT_PSI_PF 1   // changeRepr pass: next tile's words loaded into registers during this tile's layers
#endif
#define BOT_B_MAX 6   // at most layers [0, 6) run in the fused bit-sliced bottom kernel (planner: 5)

// ---------------------------------------------------------------------------------------------
// shared-memory M4R-4 lookups with the table base fused into the byte-permute that extracts the
// nibble: tables are 256-byte aligned, so PRMT(e, base, 0x7650|k) = base + (byte k of e).
// ---------------------------------------------------------------------------------------------
template <int OFF>
__device__ __forceinline__ uint32_t lds_off(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
    return v;
}

// x * c for one 32-bit limb, table tab (shared address) of constant c: XOR of 8 lookups
__device__ __forceinline__ uint32_t m4r4_word_sa(uint32_t tab, uint32_t x) {
    const uint32_t e = (x << 2) & 0x3C3C3C3Cu;   // byte k = 4 * nibble 2k
    const uint32_t o = (x >> 2) & 0x3C3C3C3Cu;   // byte k = 4 * nibble 2k+1
    uint32_t r = lds_off<0>(__byte_perm(e, tab, 0x7650));
    r ^= lds_off<64>(__byte_perm(o, tab, 0x7650));
    r ^= lds_off<128>(__byte_perm(e, tab, 0x7651));
    r ^= lds_off<192>(__byte_perm(o, tab, 0x7651));
    r ^= lds_off<256>(__byte_perm(e, tab, 0x7652));
    r ^= lds_off<320>(__byte_perm(o, tab, 0x7652));
    r ^= lds_off<384>(__byte_perm(e, tab, 0x7653));
    r ^= lds_off<448>(__byte_perm(o, tab, 0x7653));
    return r;
}
// Row t (16 words) of the M4R-4 table of constant c: tab[16t + x] = (c v_(4t)) * x, x in GF(16).
// c v_(4t) = w by SWAR products with the generators x3, x4, x5 (gf2x_device.cuh mul_v4t; no table
// lookups), and x = sum of x_b v_b (v_0 = 1, v_1 = x1, v_2 = x2, v_3 = x1 x2) so the row is the XOR-span of
// w, x1 w, x2 w, x1 x2 w.  The row's four 16-byte stores are rotated by (t >> 1): the 8 threads of a table
// (rows t = 0..7, 64 B apart) then cover all 32 banks in every store instruction (they hit 8 of them with
// 4-way conflicts in order).  (wt / SHARED: kept for the callers' signatures, unused.)
template <bool SHARED = false>
__device__ __forceinline__ void build_tab_row(uint32_t* tab, uint32_t c, int t, const uint32_t* __restrict__ wt,
                                              uint32_t* kb = nullptr) {
    (void)wt;
    const uint32_t w = mul_v4t(c, t);
    const uint32_t w1 = mulx1(w), w2 = mulx2(w), w3 = mulx1(w2);
    uint4* d = reinterpret_cast<uint4*>(tab + 16 * t);
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int qq = (q + (t >> 1)) & 3;   // entries 4 qq .. 4 qq + 3
        const uint32_t base = ((qq & 1) ? w2 : 0u) ^ ((qq & 2) ? w3 : 0u);
        d[qq] = make_uint4(base, base ^ w, base ^ w1, base ^ w ^ w1);
    }
    // small-subfield products (fft_group): K_b = c v_b, b < 8, are the entries x = 2^q of rows 0 and 1
    if (kb && t < 2) *reinterpret_cast<uint4*>(kb + 4 * t) = make_uint4(w, w1, w2, w3);
}

// ---------------------------------------------------------------------------------------------
// Multiplication by a constant c of a small subfield (Prop. 2): when c < 2^B (B = 2, 4, 8: c in
// GF(4), GF(16), GF(256), the tower's "small number => subfield" rule, definition of v_k P:658-687), every
// B-bit block of a limb is multiplied by c on its own.  The multiplier shortening puts the
// constants of layer k below 2^(m-k), so the top layers of a transform are such layers.  With
// t_b = (u >> b) & M (bit b of every block moved to the block's lowest bit, M = 0x55.., 0x11.., 0x01..),
//     c u = XOR_b t_b * (c v_b),
// each integer product t_b * K_b placing K_b = c v_b < 2^B into the blocks where bit b is set: the blocks
// are disjoint, so the integer product has no carries and equals the XOR.  IMAD runs on the FMA pipe, so
// a GF(16) product costs 9 ALU + 4 FMA-pipe instructions and no shared-memory lookup (M4R-4: 8 LDS + 15 ALU).
// ---------------------------------------------------------------------------------------------
template <int B>
__device__ __forceinline__ uint32_t smul(uint32_t u, const uint32_t* K) {
    constexpr uint32_t M = B == 2 ? 0x55555555u : (B == 4 ? 0x11111111u : 0x01010101u);
    uint32_t r = (u & M) * K[0];
#pragma unroll
    for (int b = 1; b < B; b++) r ^= ((u >> b) & M) * K[b];
    return r;
}
template <int B, bool INV>
__device__ __forceinline__ void bfly_small(uint4& x0, uint4& x1, const uint32_t* kb) {
    uint32_t K[B];
    if (B <= 4) {
        const uint4 k = *reinterpret_cast<const uint4*>(kb);
        K[0] = k.x; K[1] = k.y;
        if (B == 4) { K[2] = k.z; K[3] = k.w; }
    } else {
        const uint4 k0 = *reinterpret_cast<const uint4*>(kb), k1 = *reinterpret_cast<const uint4*>(kb + 4);
        K[0] = k0.x; K[1] = k0.y; K[2] = k0.z; K[3] = k0.w;
        K[4 % B] = k1.x; K[5 % B] = k1.y; K[6 % B] = k1.z; K[7 % B] = k1.w;
    }
    if (INV) x1 = xor4(x1, x0);
    x0.x ^= smul<B>(x1.x, K); x0.y ^= smul<B>(x1.y, K);
    x0.z ^= smul<B>(x1.z, K); x0.w ^= smul<B>(x1.w, K);
    if (!INV) x1 = xor4(x1, x0);
}

struct FftParams {
    const void* src;      // PSI: u64 novel-basis blocks (src_per per pair); else uint4 spectrum
    uint4* dst;
    const DevTables* tabs;
    uint64_t src_per;
    uint64_t batch;
    int m;                // N = 2^m points per product (local points for a shard)
    int c, k_lo, k_hi;    // tile bits [0,c) U [k_lo,k_hi)
    IdxMap map;           // local -> global index for the multipliers (identity unless sharded)
    int wt_shared;        // table builds read a shared copy of the c -> c v_(4t) maps (only where the
                          // 28 KB do not cost occupancy: the CTA holds one per SM anyway)
    int db;               // non-PSI passes: double-buffered tiles (prefetch of the next tile) if they fit
    uint4* red_dst;       // c = 5, R = 6, one product (truncated FFT, trunc.cuh): the changeRepr pass (its input)
    uint32_t red_c[6];    //   or an inverse pass (its output) also folds the tile's 6 index bits [k_lo, k_hi)
                          //   with the Reduce constants red_c[k - k_lo] into red_dst[base | col]
    int st_tma;           // double-buffered non-PSI passes: tiles leave by one TMA tensor store (map over dst)
    int ld_tma;           // (with st_tma) and arrive by one TMA tensor load (map over src)
};

// x[u] ^= c x[u + HALF], u < HALF (one Reduce level in registers; tl = the M4R-4 table of c)
template <int HALF>
__device__ __forceinline__ void reduce_level(uint4* x, uint32_t tl) {
#pragma unroll
    for (int u = 0; u < HALF; u++) {
        const uint4 v = x[u + HALF];
        x[u].x ^= m4r4_word_sa(tl, v.x); x[u].y ^= m4r4_word_sa(tl, v.y);
        x[u].z ^= m4r4_word_sa(tl, v.z); x[u].w ^= m4r4_word_sa(tl, v.w);
    }
}

__device__ __forceinline__ uint32_t tab_addr(uint32_t base, uint32_t id) { return base + id * 512u; }

template <bool INV>
__device__ __forceinline__ void bfly(uint4& x0, uint4& x1, uint32_t ta) {
    if (!INV) {
        x0.x ^= m4r4_word_sa(ta, x1.x); x0.y ^= m4r4_word_sa(ta, x1.y);
        x0.z ^= m4r4_word_sa(ta, x1.z); x0.w ^= m4r4_word_sa(ta, x1.w);
        x1 = xor4(x1, x0);
    } else {
        x1 = xor4(x1, x0);
        x0.x ^= m4r4_word_sa(ta, x1.x); x0.y ^= m4r4_word_sa(ta, x1.y);
        x0.z ^= m4r4_word_sa(ta, x1.z); x0.w ^= m4r4_word_sa(ta, x1.w);
    }
}

// One group of r consecutive layers [ka, ka+r) whose slot bits are [s0, s0+r).
// Table id of (layer k, slot) = 2^(R-1-kk) - 1 + (row >> (kk+1)), row = slot >> c, kk = k - k_lo.
// A layer whose constants lie in GF(4) / GF(16) (/ GF(256) with FFT_SMALL_MAX 8) -- global layer kg of a
// transform over at most 2^mg global indices has constants < 2^(mg - kg) -- multiplies by bfly_small.
#ifndef FFT_SMALL_MAX
#define FFT_SMALL_MAX 4
#endif
template <int r, bool INV, bool ZS>
__device__ __forceinline__ void fft_group(uint4* tile, uint32_t nslots, int s0, int ka, const FftParams& p, uint32_t tabs_sa,
                                          const uint32_t* zf, const uint32_t* kbt) {
    const uint32_t nitems = nslots >> r;
    const int R = p.k_hi - p.k_lo;
    const int mg = p.m + p.map.bits;
    uint32_t it = threadIdx.x;
    for (; it < nitems; it += blockDim.x) {
        const uint32_t base = (it & ((1u << s0) - 1)) | ((it >> s0) << (s0 + r));
        uint4 v[1 << r];
#pragma unroll
        for (int j = 0; j < (1 << r); j++) v[j] = tile[base | ((uint32_t)j << s0)];
#pragma unroll
        for (int li = 0; li < r; li++) {
            const int lb = INV ? li : (r - 1 - li);   // local bit of this layer
            const int kk = ka + lb - p.k_lo;
            const int wbits = mg - glayer(p.map, ka + lb);   // the layer's constants are < 2^wbits
            // (only passes holding the top layer (ZS) have such layers in the single-GPU plans; the others keep
            // one code path: measured 6 % slower with the class test compiled into every pass)
            const int cls = !ZS ? 0 : (wbits <= 2 ? 2 : (wbits <= 4 ? 4 : (wbits <= FFT_SMALL_MAX ? 8 : 0)));
            if (cls == 0) {
#pragma unroll
                for (int j = 0; j < (1 << r); j++) {
                    if (j & (1 << lb)) continue;
                    const uint32_t row = (base | ((uint32_t)j << s0)) >> p.c;
                    const uint32_t id = ((1u << (R - 1 - kk)) - 1) + (row >> (kk + 1));
                    // multiplier 0 (the block at base 0: s_k vanishes on V_k, Claim 1 P:696-701): x1 ^= x0 only
                    // (warp-uniform branch; a third of the first forward / last inverse pass)
                    if (ZS && zf[id]) v[j | (1 << lb)] = xor4(v[j | (1 << lb)], v[j]);
                    else bfly<INV>(v[j], v[j | (1 << lb)], tab_addr(tabs_sa, id));
                }
            } else {
#pragma unroll
                for (int j = 0; j < (1 << r); j++) {
                    if (j & (1 << lb)) continue;
                    const uint32_t row = (base | ((uint32_t)j << s0)) >> p.c;
                    const uint32_t id = ((1u << (R - 1 - kk)) - 1) + (row >> (kk + 1));
                    const uint32_t* kb = kbt + id * 8;
                    if (cls == 2) bfly_small<2, INV>(v[j], v[j | (1 << lb)], kb);
                    else if (cls == 4) bfly_small<4, INV>(v[j], v[j | (1 << lb)], kb);
                    else bfly_small<(FFT_SMALL_MAX >= 8 ? 8 : 4), INV>(v[j], v[j | (1 << lb)], kb);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < (1 << r); j++) tile[base | ((uint32_t)j << s0)] = v[j];
    }
}

template <bool INV, bool ZS>
__device__ __forceinline__ void fft_group_any(int r, uint4* tile, uint32_t nslots, int s0, int ka, const FftParams& p,
                                              uint32_t tabs_sa, const uint32_t* zf, const uint32_t* kbt) {
    if (r == 3) fft_group<3, INV, ZS>(tile, nslots, s0, ka, p, tabs_sa, zf, kbt);
    else if (r == 2) fft_group<2, INV, ZS>(tile, nslots, s0, ka, p, tabs_sa, zf, kbt);
    else fft_group<1, INV, ZS>(tile, nslots, s0, ka, p, tabs_sa, zf, kbt);
}

// shared memory: [tables (2^R - 1) x 512 B] [psi table (PSI)] [tile]
#ifndef FFT_MINB
#define FFT_MINB 2
#endif
// ZS: the pass holds the top layer (k_hi = m), where the multiplier-0 blocks are a large share
template <bool INV, bool PSI, bool ZS>
__global__ void __launch_bounds__(FFT_THREADS, FFT_MINB) k_fft2(FftParams p, const __grid_constant__ CUtensorMap tm,
                                                                const __grid_constant__ CUtensorMap tm_src) {
    __shared__ __align__(8) uint64_t fbars[2];   // (p.ld_tma) TMA tile loads, one mbarrier per buffer
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int R = p.k_hi - p.k_lo;
    const uint32_t nslots = 1u << (p.c + R);
    const uint32_t ntab = (1u << R) - 1;
    // shared memory: [tables (ntab x 512 B)] [psi table (PSI)] [zero flags, 512 B] [wt copy, 28 KB] [tile]
    // [second tile (!PSI)]
    uint32_t* tabs = reinterpret_cast<uint32_t*>(smem_raw);
    uint4* psit = reinterpret_cast<uint4*>(tabs + ntab * 128);
    uint32_t* zf = reinterpret_cast<uint32_t*>(psit + (PSI ? 8 * 256 : 0));   // per table: multiplier == 0
    uint32_t* kbt = zf + 128;                                                   // per table: K_b = c v_b, b < 8
    uint32_t* wts = kbt + 128 * 8;                                              // M4R-8 maps c -> c v_(4t)
    const uint32_t tile_off = (uint32_t)(ntab * 512 + (PSI ? 8 * 256 * 16 : 0) + 512 + 4096 + (p.wt_shared ? 7 * 1024 * 4 : 0));
    uint4* tile = reinterpret_cast<uint4*>(smem_raw + tile_off);
    const uint32_t tabs_sa = (uint32_t)__cvta_generic_to_shared(tabs);
    if (tabs_sa & 255) __trap();  // the PRMT address fusion needs 256-byte aligned tables
    if (PSI)
        for (uint32_t i = threadIdx.x; i < 8 * 256; i += blockDim.x) psit[i] = p.tabs->psi64[i];
    if (p.wt_shared)
        for (uint32_t i = threadIdx.x; i < 7 * 1024 / 4; i += blockDim.x)
            reinterpret_cast<uint4*>(wts)[i] = reinterpret_cast<const uint4*>(p.tabs->wt)[i];
    // fused Reduce (the forward changeRepr pass: of its input tile; the last inverse pass: of its output tile):
    // 6 tables after the tile(s), then an 8 x 32 scratch
    uint32_t* rtab = reinterpret_cast<uint32_t*>(smem_raw + tile_off + nslots * 16 * ((!PSI && p.db) ? 2 : 1));
    uint4* rscr = reinterpret_cast<uint4*>(rtab + 6 * 128);
    // Reduce over slot bits [5, 11) (index bits [k_lo, k_hi)): thread (part, col) folds u = 8 part + v over v's
    // bits, then 32 threads fold the 8 parts; the tile itself is only read
    auto fold_tile = [&](uint32_t base) {
        const uint32_t rt = (uint32_t)__cvta_generic_to_shared(rtab);
        const uint32_t col = threadIdx.x & 31, part = threadIdx.x >> 5;
        uint4 x[8];
#pragma unroll
        for (int v = 0; v < 8; v++) x[v] = tile[col | ((part * 8 + v) << 5)];
        reduce_level<4>(x, rt + 512 * 2);
        reduce_level<2>(x, rt + 512 * 1);
        reduce_level<1>(x, rt);
        rscr[part * 32 + col] = x[0];
        __syncthreads();
        if (threadIdx.x < 32) {
#pragma unroll
            for (int q = 0; q < 8; q++) x[q] = rscr[q * 32 + threadIdx.x];
            reduce_level<4>(x, rt + 512 * 5);
            reduce_level<2>(x, rt + 512 * 4);
            reduce_level<1>(x, rt + 512 * 3);
            p.red_dst[base | threadIdx.x] = x[0];
        }
    };
    if ((PSI || INV) && p.red_dst && threadIdx.x < 48) {
        const int l = threadIdx.x >> 3;
        uint32_t cst = p.red_c[0];
#pragma unroll
        for (int q = 1; q < 6; q++) cst = l == q ? p.red_c[q] : cst;
        build_tab_row(rtab + 128 * l, cst, threadIdx.x & 7, p.tabs->wt);
    }
    // TMA tile loads (p.ld_tma, with p.st_tma, double-buffered non-PSI passes): thread 0 loads a tile with one 4-D
    // tensor load (the store's geometry over src), completing on the buffer's mbarrier
    const bool ldm = !PSI && p.db && p.st_tma && p.ld_tma;
    if (ldm && threadIdx.x == 0) {
        mbar_init(&fbars[0], 1);
        mbar_init(&fbars[1], 1);
        mbar_fence_init();
    }
    __syncthreads();   // the first tile's table build / load reads entries other warps wrote

    const uint64_t N = 1ull << p.m;
    const uint64_t tiles_per_pair = N >> (p.c + R);
    const uint64_t ntiles = tiles_per_pair * p.batch;
    const uint32_t cmask = (1u << p.c) - 1;

    const int midbits = p.k_lo - p.c;
    // base index (within the pair) of tile t: bits [c, k_lo) and >= k_hi come from tt
    auto tile_geom = [&](uint64_t t, uint64_t& pair, uint32_t& base) {
        pair = t / tiles_per_pair;
        const uint32_t tt = (uint32_t)(t - pair * tiles_per_pair);
        base = ((tt & ((1u << midbits) - 1)) << p.c) | ((uint32_t)((uint64_t)(tt >> midbits) << p.k_hi));
    };
    // Each CTA takes a contiguous run of tiles: consecutive tiles differ in the column/middle index bits
    // [c, k_lo) first, which no multiplier of the pass depends on (layer k >= k_lo uses bits > k), so the
    // tables are rebuilt only when the bits >= k_hi change (rarely in the upper passes).
    const uint64_t per_cta = ntiles / gridDim.x, extra = ntiles % gridDim.x;
    const uint64_t t_begin = blockIdx.x * per_cta + min((uint64_t)blockIdx.x, extra);
    const uint64_t t_end = t_begin + per_cta + (blockIdx.x < extra ? 1 : 0);
    // non-PSI passes are double-buffered: the next tile is prefetched with cp.async during this one
    auto prefetch = [&](uint64_t t, uint32_t off) {
        uint64_t pair; uint32_t base;
        tile_geom(t, pair, base);
        const uint4* src = reinterpret_cast<const uint4*>(p.src) + pair * N;
        uint4* buf = reinterpret_cast<uint4*>(smem_raw + off);
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x)
            cp_async16(buf + s, src + (base | (s & cmask) | ((s >> p.c) << p.k_lo)));
    };
    const uint32_t tbytes = nslots * 16;
    auto tma_prefetch = [&](uint64_t t, int b) {   // thread 0 only
        uint64_t pair; uint32_t base;
        tile_geom(t, pair, base);
        const uint64_t tt = t - pair * tiles_per_pair;
        mbar_arrive_expect_tx(&fbars[b], tbytes);
        tma_load_4d(smem_raw + tile_off + b * tbytes, &tm_src, 0, (int)(tt & ((1u << midbits) - 1)), 0,
                    (int)(pair * (N >> p.k_hi) + (tt >> midbits)), &fbars[b]);
    };
    if (ldm) {
        if (threadIdx.x == 0 && t_begin < t_end) tma_prefetch(t_begin, 0);
    } else if (!PSI && p.db) {
        if (t_begin < t_end) prefetch(t_begin, tile_off);
        cp_async_commit();
    }
    int kt = 0;
    uint32_t tab_key = 0xFFFFFFFFu;
    // TMA stores (p.st_tma, double-buffered non-PSI passes): thread 0 stores the finished tile with one 4-D tensor
    // store (dims: the 2^c-unit column run, middle bits [c, k_lo), rows [k_lo, k_hi), the rest incl. pairs); the
    // next tile's prefetch into the other buffer is issued after the first layer group, once that store has read
    // it (cp.async.bulk.wait_group.read)
    // (the single-buffered PSI pass: the next tile's changeRepr writes wait for the store to have read the tile)
    const bool stm = p.st_tma && (PSI || p.db);
    // PSI passes whose tile is one FFT_UNR-word batch per thread: the next tile's words are loaded into registers
    // before this tile's layers (software pipelining; the pass has no room for a second tile buffer)
    // (also tiles of fewer slots, e.g. one 2^9-point product of a batch: nslots / threads words per thread)
    const bool psi_pf = PSI && FFT_PSI_PF && nslots <= (uint32_t)FFT_UNR * blockDim.x && nslots % blockDim.x == 0;
    uint64_t wn[FFT_UNR];
    auto psi_load = [&](uint64_t tt, uint64_t* w) {
        uint64_t pair; uint32_t base;
        tile_geom(tt, pair, base);
        const uint64_t* src = reinterpret_cast<const uint64_t*>(p.src) + pair * p.src_per;
#pragma unroll
        for (int u = 0; u < FFT_UNR; u++) {
            const uint32_t s = threadIdx.x + u * blockDim.x;
            const uint32_t g = base | (s & cmask) | ((s >> p.c) << p.k_lo);
            w[u] = (s < nslots && g < p.src_per) ? src[g] : 0ull;
        }
    };
    if (psi_pf && t_begin < t_end) psi_load(t_begin, wn);
    for (uint64_t t = t_begin; t < t_end; t++, kt++) {
        uint64_t pair;
        uint32_t base;
        tile_geom(t, pair, base);
        if (!PSI) {
            if (p.db) {
                tile = reinterpret_cast<uint4*>(smem_raw + tile_off + (kt & 1) * tbytes);
                if (!stm && t + 1 < t_end) prefetch(t + 1, tile_off + ((kt + 1) & 1) * tbytes);
            } else {
                prefetch(t, tile_off);   // single buffer: this tile's copies, waited for below
            }
            if (!ldm) cp_async_commit();
        }
        // ---- tables of this tile's multipliers: id -> (layer kk, block blk); they depend on base >> k_hi only
        const uint32_t key = (uint32_t)((uint64_t)base >> p.k_hi);
        if (key != tab_key)
        for (uint32_t i = threadIdx.x; i < ntab * 8; i += blockDim.x) {
            const uint32_t id = i >> 3;
            const int lg = 31 - __clz(id + 1);          // = R-1-kk
            const int k = p.k_lo + R - 1 - lg;
            const uint32_t blk = id + 1 - (1u << lg);
            const uint32_t lb = (uint32_t)(((uint64_t)base & ~((2ull << k) - 1)) | ((uint64_t)blk << (k + 1)));
            const uint32_t cst = layer_const(glayer(p.map, k), gidx(p.map, lb));
            uint32_t* kbo = ZS ? kbt + id * 8 : nullptr;
            if (p.wt_shared) build_tab_row<true>(tabs + id * 128, cst, (int)(i & 7), wts, kbo);
            else build_tab_row<false>(tabs + id * 128, cst, (int)(i & 7), p.tabs->wt, kbo);
            if ((i & 7) == 0) zf[id] = cst == 0;
        }
        tab_key = key;
        // ---- load
        if (PSI && stm && kt > 0) {
            if (threadIdx.x == 0) bulk_wait_read<0>();
            __syncthreads();
        }
        if (PSI) {
            // FFT_UNR loads in flight per thread, then changeRepr of each word (M4R-8, 8 lookups)
            const uint64_t* src = reinterpret_cast<const uint64_t*>(p.src) + pair * p.src_per;
            for (uint32_t s0 = threadIdx.x; s0 < nslots; s0 += FFT_UNR * blockDim.x) {
                uint64_t w[FFT_UNR];
                if (psi_pf) {
#pragma unroll
                    for (int u = 0; u < FFT_UNR; u++) w[u] = wn[u];
                } else {
#pragma unroll
                    for (int u = 0; u < FFT_UNR; u++) {
                        const uint32_t s = s0 + u * blockDim.x;
                        const uint32_t g = base | (s & cmask) | ((s >> p.c) << p.k_lo);
                        w[u] = (s < nslots && g < p.src_per) ? src[g] : 0ull;
                    }
                }
#pragma unroll
                for (int u = 0; u < FFT_UNR; u++) {
                    const uint32_t s = s0 + u * blockDim.x;
                    uint4 v = make_uint4(0, 0, 0, 0);
                    if (w[u]) {
#pragma unroll
                        for (int ch = 0; ch < 8; ch++) v = xor4(v, psit[ch * 256 + ((w[u] >> (8 * ch)) & 255)]);
                    }
                    if (s < nslots) tile[s] = v;
                }
            }
        } else {
            if (ldm) mbar_wait(&fbars[kt & 1], (uint32_t)(kt >> 1) & 1);
            else if (p.db) cp_async_wait<1>();   // this tile's copies have landed (the next tile's may be in flight)
            else cp_async_wait<0>();
        }
        if (psi_pf && t + 1 < t_end) psi_load(t + 1, wn);   // in flight during this tile's layers
        __syncthreads();
        if (!INV && PSI && p.red_dst) fold_tile(base);
        // ---- layers, in groups of <= 3 (forward: from the top; inverse: from the bottom)
        bool first = true;
        auto after_group = [&]() {   // (stm) the previous store has read the other buffer: refill it
            if (!PSI && stm && first && threadIdx.x == 0) {
                bulk_wait_read<0>();
                if (ldm && t + 1 < t_end) tma_prefetch(t + 1, (kt + 1) & 1);
            }
            __syncthreads();
            if (!PSI && stm && first && !ldm) {
                if (t + 1 < t_end) prefetch(t + 1, tile_off + ((kt + 1) & 1) * tbytes);
                cp_async_commit();
            }
            first = false;
        };
        if (!INV) {
            int top = p.k_hi;
            while (top > p.k_lo) {
                const int r = (top - p.k_lo) >= 3 ? 3 : (top - p.k_lo);
                const int ka = top - r;
                fft_group_any<INV, ZS>(r, tile, nslots, p.c + ka - p.k_lo, ka, p, tabs_sa, zf, kbt);
                after_group();
                top = ka;
            }
        } else {
            int bot = p.k_lo;
            while (bot < p.k_hi) {
                const int r = (p.k_hi - bot) >= 3 ? 3 : (p.k_hi - bot);
                fft_group_any<INV, ZS>(r, tile, nslots, p.c + bot - p.k_lo, bot, p, tabs_sa, zf, kbt);
                after_group();
                bot += r;
            }
        }
        if (INV && p.red_dst) fold_tile(base);
        // ---- store
        if (stm) {
            fence_proxy_async_smem();   // the layers' writes before the tensor store's reads
            __syncthreads();
            if (threadIdx.x == 0) {
                const uint64_t tt = t - pair * tiles_per_pair;
                tma_store_4d(&tm, 0, (int)(tt & ((1u << midbits) - 1)), 0, (int)(pair * (N >> p.k_hi) + (tt >> midbits)), tile);
                bulk_commit();
            }
            continue;
        }
        uint4* dst = p.dst + pair * N;
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x) dst[base | (s & cmask) | ((s >> p.c) << p.k_lo)] = tile[s];
        __syncthreads();
    }
    if (!PSI) cp_async_wait<0>();
    if (stm && threadIdx.x == 0) bulk_wait<0>();
}

static size_t fft2_smem(int c, int R, bool psi, bool wt_shared, bool db, bool red = false) {
    size_t s = red ? 6 * 512 + 8 * 32 * 16 : 0;
    s += (((size_t)1 << R) - 1) * 512;
    if (psi) s += 8 * 256 * 16;
    s += 512;   // zero-multiplier flags (<= 127 tables)
    s += 4096;  // small-subfield constants K_b (<= 127 tables x 8 words)
    if (wt_shared) s += 7 * 1024 * 4;   // shared copy of the M4R-8 maps c -> c v_(4t) (table builds)
    s += ((size_t)1 << (c + R)) * 16 * (db ? 2 : 1);
    return s;
}
// non-psi passes are double-buffered when two tiles fit
static bool fft2_db(int c, int R, bool psi) { return !psi && fft2_smem(c, R, psi, false, true) <= 200 * 1024; }
// the shared wt copy only where the CTA already takes a whole SM (it would otherwise halve occupancy)
static bool fft2_wt_shared(int c, int R, bool psi) {
    (void)c; (void)R; (void)psi;
    return false;   // the table rows are built by SWAR products (build_tab_row): no c -> c v_(4t) maps needed
}
