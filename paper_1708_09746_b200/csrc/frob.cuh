// frob.cuh -- App. C building block: BasisCvt / iBasisCvt on GF(2)
// coefficients ("The basis conversion can be proceeded straightforwardly with alg. 3"), the first
// step of the multiply through the Frobenius bijection.  Included by gf2x.cu.
//
// The coefficients are packed 64 per word (bit t of the polynomial = bit t % 64 of word t / 64).  Alg. 3's
// Taylor steps (Alg. 2, the same (lg, K) list as the word-level conversion, in the paper's order) act on
// bit positions: step (lg, K) on every segment of 2^lg bits, h = 2^(lg-1), u = h >> K,
// d = h - u, "f[i - d] ^= f[i] for i = 2h-1 .. h" splits into two parallel sweeps (the targets of one sweep
// are never its sources):
//   sweep 1: targets [h, h + u)  (sources [2h - u, 2h));   sweep 2: targets [u, h)  (sources [h, 2h - u)),
// forward in the order 1, 2 and inverse (ascending i) in the order 2, 1.  One thread owns one word: it
// XORs in the source bits (a funnel shift of the words d bits up) under the mask of its target bits; words
// that hold no targets are not touched.  This is the plain form of the step (one HBM sweep each); the tiled
// forms of the word-level conversion are the next step for it.
#pragma once

// lg >= 7: only the words that hold targets are visited (ntw of every segment of 2^(lg-6) words)
__global__ void __launch_bounds__(256) k_bitcvt_sweep(uint64_t* __restrict__ G, uint64_t nw, int lg, uint64_t d,
                                                      uint64_t tlo, uint64_t thi) {
    const uint64_t len = 1ull << lg, wps = len >> 6, tw0 = tlo >> 6, ntw = ((thi + 63) >> 6) - tw0;
    const uint64_t total = (nw / wps) * ntw;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t seg = t / ntw, w = seg * wps + tw0 + (t - seg * ntw);
        const uint64_t o = (w << 6) & (len - 1);   // the word's offset in its segment
        const uint64_t lo = tlo > o ? tlo - o : 0, hi = thi < o + 64 ? thi - o : 64;
        if (lo >= hi) continue;
        const uint64_t mask = (hi >= 64 ? ~0ull : ((1ull << hi) - 1)) & ~((1ull << lo) - 1);
        const uint64_t sp = (w << 6) + d, w0 = sp >> 6;
        const int sh = (int)(sp & 63);
        uint64_t src = G[w0] >> sh;
        if (sh && w0 + 1 < nw) src |= G[w0 + 1] << (64 - sh);
        G[w] ^= src & mask;
    }
}

// a run of steps whose segments lie inside one word (lg <= 6), applied to every word in registers
struct InwordSweeps {
    uint64_t pmask[64];
    int d[64];
    int n;
};
__global__ void __launch_bounds__(256) k_bitcvt_inword(uint64_t* __restrict__ G, uint64_t nw, InwordSweeps sw) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = G[w];
        for (int k = 0; k < sw.n; k++) x ^= (x >> sw.d[k]) & sw.pmask[k];
        G[w] = x;
    }
}

// The inner conversion BasisCvt_C(q_i) of every 2^C-bit chunk (C <= 16: 8 KB) in one pass through shared
// memory: the chunk's words are loaded once and all its sweeps (in-word, across bit 6 and word-aligned alike)
// run on them with a barrier after each.
#define BITCHUNK_MAXSW 96
struct ChunkSweeps {
    uint64_t pmask[BITCHUNK_MAXSW];   // lg <= 6: periodic target mask
    uint32_t d[BITCHUNK_MAXSW], tlo[BITCHUNK_MAXSW], thi[BITCHUNK_MAXSW];
    uint8_t lg[BITCHUNK_MAXSW];
    int n, cw;                        // sweeps; words per chunk (2^(C-6))
};
// sweeps [k0, k1) of a chunk held in shared memory (a barrier after each sweep or in-word run)
__device__ __forceinline__ void chunk_sweeps(uint64_t* T, uint32_t cw, const ChunkSweeps& sw, int k0, int k1) {
    for (int k = k0; k < k1; k++) {
        const int lg = sw.lg[k];
        const uint32_t d = sw.d[k];
        if (lg <= 6) {
            // a run of consecutive in-word sweeps: each thread applies all of them to its own words in
            // registers (no word is read by another thread), with one barrier after the run
            int kr = k + 1;
            while (kr < k1 && sw.lg[kr] <= 6) kr++;
            for (uint32_t w = threadIdx.x; w < cw; w += blockDim.x) {
                uint64_t x = T[w];
                for (int q = k; q < kr; q++) x ^= (x >> sw.d[q]) & sw.pmask[q];
                T[w] = x;
            }
            k = kr - 1;
        } else {
            const uint32_t tlo = sw.tlo[k], thi = sw.thi[k], len = 1u << lg, wps = len >> 6, tw0 = tlo >> 6;
            const uint32_t ntw = ((thi + 63) >> 6) - tw0, total = (cw / wps) * ntw;
            uint64_t nv[4];
            uint32_t nwd[4];
            int cnt = 0;
            // read phase (all sources first: a target word may be another thread's source word)
            for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
                const uint32_t seg = t / ntw, w = seg * wps + tw0 + (t - seg * ntw);
                const uint32_t o = (w << 6) & (len - 1);
                const uint32_t lo = tlo > o ? tlo - o : 0, hi = thi < o + 64 ? thi - o : 64;
                if (lo >= hi) continue;
                const uint64_t mask = (hi >= 64 ? ~0ull : ((1ull << hi) - 1)) & ~((1ull << lo) - 1);
                const uint32_t sp = (w << 6) + d, w0 = sp >> 6, sh = sp & 63;
                uint64_t src = T[w0] >> sh;
                if (sh && w0 + 1 < cw) src |= T[w0 + 1] << (64 - sh);
                nv[cnt] = T[w] ^ (src & mask);
                nwd[cnt++] = w;
            }
            __syncthreads();
            for (int q = 0; q < cnt; q++) T[nwd[q]] = nv[q];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_bitcvt_chunk(uint64_t* __restrict__ G, uint64_t nchunks, ChunkSweeps sw) {
    __shared__ uint64_t T[1024];
    const uint32_t cw = (uint32_t)sw.cw;
    for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        uint64_t* g = G + ch * cw;
        __syncthreads();
        for (uint32_t w = threadIdx.x; w < cw; w += blockDim.x) T[w] = g[w];
        __syncthreads();
        chunk_sweeps(T, cw, sw, 0, sw.n);
        for (uint32_t w = threadIdx.x; w < cw; w += blockDim.x) g[w] = T[w];
    }
}

// ---- 2^16-bit chunks (C = 16, the c4a / c4b case) with their inner blocks in registers.  bit_ops(16) =
// [levels 16..9, K = 8][bit_ops(8, 8): levels 16..13 (K = 4), then bit_ops(4, 12), bit_ops(4, 8)]
// [bit_ops(8, 0)].  bit_ops(4, 12) and bit_ops(4, 8) are the 16-unit network of cvt_ops(4) (cvt16_regs,
// small.cuh: the same steps, its last two in the other order -- they act on disjoint index bits and commute,
// R26) on 16 words at stride 64 and at stride 4; bit_ops(8, 0) acts inside every 256-bit window (4 words): one
// thread applies its 12 steps to a window as 256-bit shift-mask-XOR operations with compile-time constants.
// The top run and levels 16..13 stay shared-memory sweeps (ChunkSweeps, 24 of them).
constexpr uint64_t bw_mask(int lg, int K, bool A, int wi) {   // word wi of the step's target mask in 256 bits
    uint64_t m = 0;
    for (int b = 0; b < 64; b++) {
        const int t = (wi * 64 + b) & ((1 << lg) - 1), h = 1 << (lg - 1), u = h >> K;
        if (A ? (t >= h && t < h + u) : (t >= u && t < h)) m |= 1ull << b;
    }
    return m;
}
template <int LG, int K, bool A>
__device__ __forceinline__ void bw_sweep(uint64_t* x) {   // x ^= (x >> d) & mask on 256 bits
    constexpr int d = (1 << (LG - 1)) - ((1 << (LG - 1)) >> K), q = d >> 6, r = d & 63;
    uint64_t y[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        uint64_t v = i + q < 4 ? x[i + q] >> r : 0ull;
        if (r && i + q + 1 < 4) v |= x[i + q + 1] << (64 - r);
        y[i] = v;
    }
    x[0] ^= y[0] & bw_mask(LG, K, A, 0);
    x[1] ^= y[1] & bw_mask(LG, K, A, 1);
    x[2] ^= y[2] & bw_mask(LG, K, A, 2);
    x[3] ^= y[3] & bw_mask(LG, K, A, 3);
}
template <int LG, int K, bool INV>
__device__ __forceinline__ void bw_step(uint64_t* x) {
    bw_sweep<LG, K, !INV>(x);
    bw_sweep<LG, K, INV>(x);
}
// bit_ops(8, 0) in the paper's order: (8,4) (7,4) (6,4) (5,4) (8,2) (7,2) (8,1) (6,1) (4,2) (3,2) (4,1) (2,1)
template <bool INV>
__device__ __forceinline__ void bw_cvt256(uint64_t* x) {
    if (!INV) {
        bw_step<8, 4, false>(x); bw_step<7, 4, false>(x); bw_step<6, 4, false>(x); bw_step<5, 4, false>(x);
        bw_step<8, 2, false>(x); bw_step<7, 2, false>(x); bw_step<8, 1, false>(x); bw_step<6, 1, false>(x);
        bw_step<4, 2, false>(x); bw_step<3, 2, false>(x); bw_step<4, 1, false>(x); bw_step<2, 1, false>(x);
    } else {
        bw_step<2, 1, true>(x); bw_step<4, 1, true>(x); bw_step<3, 2, true>(x); bw_step<4, 2, true>(x);
        bw_step<6, 1, true>(x); bw_step<8, 1, true>(x); bw_step<7, 2, true>(x); bw_step<8, 2, true>(x);
        bw_step<5, 4, true>(x); bw_step<6, 4, true>(x); bw_step<7, 4, true>(x); bw_step<8, 4, true>(x);
    }
}
template <bool INV>
__global__ void __launch_bounds__(256) k_bitcvt_chunk16(uint64_t* __restrict__ G, uint64_t nchunks, ChunkSweeps sw) {
    __shared__ uint64_t T[1024];
    const uint32_t tid = threadIdx.x;
    for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        uint64_t* g = G + ch * 1024;
        __syncthreads();
        for (uint32_t w = tid; w < 1024; w += blockDim.x) T[w] = g[w];
        __syncthreads();
        if (!INV) chunk_sweeps(T, 1024, sw, 0, sw.n);   // levels 16..9 and 16..13
        for (int ph = 0; ph < 3; ph++) {
            // forward: bit_ops(4, 12), bit_ops(4, 8), bit_ops(8, 0); inverse: the reverse
            const int f = INV ? 2 - ph : ph;
            if (f == 0) { if (tid < 64) cvt16_pass<uint64_t, INV>(T, tid, 64); }
            else if (f == 1) { if (tid < 64) cvt16_pass<uint64_t, INV>(T, (tid >> 2) * 64 + (tid & 3), 4); }
            else {
                uint64_t x[4];
#pragma unroll
                for (int i = 0; i < 4; i++) x[i] = T[tid * 4 + i];
                bw_cvt256<INV>(x);
#pragma unroll
                for (int i = 0; i < 4; i++) T[tid * 4 + i] = x[i];
            }
            __syncthreads();
        }
        if (INV) chunk_sweeps(T, 1024, sw, 0, sw.n);
        for (uint32_t w = tid; w < 1024; w += blockDim.x) g[w] = T[w];
    }
}

// Alg. 3's steps in the paper's order (Taylor levels, outer conversion, inner conversions; the oracle's order)
static void bit_ops(int m, int sigma, std::vector<CvtOp>& out) {
    if (m <= 1) return;
    int K = 1;
    while (2 * K <= m - 1) K *= 2;
    for (int l = m; l >= K + 1; --l) out.push_back({l + sigma, K});
    bit_ops(m - K, sigma + K, out);
    bit_ops(K, sigma, out);
}

// A step whose window [lg-1-K, lg) of index bits lies at or above bit 6 moves whole words: consecutive such
// steps run as a word-level conversion (the planned res / rb / tile passes of the Alg. 5 path on the packed
// words, step (lg - 6, K)); steps inside a word fuse into one in-register pass; the rest (windows across bit 6)
// are bit sweeps.
static void bit_sweeps(const CvtOp& op, bool inverse, ChunkSweeps& cs) {
    const uint64_t h = 1ull << (op.lg - 1), u = h >> op.K, d = h - u;
    for (int sw = 0; sw < 2; sw++) {
        const bool first = inverse ? sw == 1 : sw == 0;
        const uint64_t tlo = first ? h : u, thi = first ? h + u : h;
        uint64_t pmask = 0;
        if (op.lg <= 6)
            for (uint64_t seg = 0; seg < 64; seg += 2 * h)
                for (uint64_t t = tlo; t < thi; t++) pmask |= 1ull << (seg + t);
        const int k = cs.n++;
        cs.pmask[k] = pmask; cs.d[k] = (uint32_t)d; cs.tlo[k] = (uint32_t)tlo; cs.thi[k] = (uint32_t)thi; cs.lg[k] = (uint8_t)op.lg;
    }
}

static gf2x_status run_bitcvt(uint64_t* G, int M, bool inverse, int smc, cudaStream_t st) {
    // the inner conversions of the 2^C-bit chunks (C = the top level's K, or all of it for M <= 16) go to
    // k_bitcvt_chunk; they come last in the paper's order (first when inverse)
    int C = M;
    if (M > 16) { C = 1; while (2 * C <= M - 1) C *= 2; }
    const bool chunked = C >= 7 && C <= 16 && !env_flag("GF2X_BITCVT_NOCHUNK");
    std::vector<CvtOp> ops;
    if (chunked && C < M) {   // top Taylor levels and the outer conversion of the top node
        for (int l = M; l >= C + 1; --l) ops.push_back({l, C});
        bit_ops(M - C, C, ops);
    } else if (!chunked) {
        bit_ops(M, 0, ops);
    }
    auto run_chunks = [&]() -> gf2x_status {
        std::vector<CvtOp> inner;
        bit_ops(C, 0, inner);
        // C = 16: only the top run and levels 16..13 as sweeps, the rest in registers (k_bitcvt_chunk16); the
        // kernel's fixed inner lists are checked against bit_ops here
        const bool c16 = C == 16 && !env_flag_now("GF2X_BITCVT_NOREG");
        if (c16) {
            std::vector<CvtOp> hi, lo, want;
            bit_ops(4, 12, hi);
            bit_ops(4, 8, hi);
            bit_ops(8, 0, lo);
            const int ref[12][2] = {{8, 4}, {7, 4}, {6, 4}, {5, 4}, {8, 2}, {7, 2}, {8, 1}, {6, 1}, {4, 2}, {3, 2}, {4, 1}, {2, 1}};
            bool ok = inner.size() == 12 + hi.size() + lo.size() && lo.size() == 12;
            for (size_t i = 0; ok && i < hi.size(); i++)
                ok = inner[12 + i].lg == hi[i].lg && inner[12 + i].K == hi[i].K && hi[i].K <= 2;
            for (int i = 0; ok && i < 12; i++) ok = lo[i].lg == ref[i][0] && lo[i].K == ref[i][1] && inner[12 + hi.size() + i].lg == lo[i].lg;
            if (!ok) return fail(GF2X_EINVAL, "bit-level chunk: unexpected inner op list");
            inner.resize(12);   // levels 16..9 (K = 8) and 16..13 (K = 4)
        }
        if (inverse) std::reverse(inner.begin(), inner.end());
        ChunkSweeps cs;
        cs.n = 0;
        cs.cw = 1 << (C - 6);
        for (const CvtOp& op : inner) {
            if (cs.n + 2 > BITCHUNK_MAXSW) return fail(GF2X_EINVAL, "bit-level chunk: too many sweeps");
            bit_sweeps(op, inverse, cs);
        }
        const uint64_t nchunks = (1ull << (M - 6)) >> (C - 6);
        ProfScope ps("k_bitcvt_chunk", 16.0 * (double)(1ull << (M - 6)), st);
        if (c16 && inverse) k_bitcvt_chunk16<true><<<grid_for(nchunks, 1, smc, 8), 256, 0, st>>>(G, nchunks, cs);
        else if (c16) k_bitcvt_chunk16<false><<<grid_for(nchunks, 1, smc, 8), 256, 0, st>>>(G, nchunks, cs);
        else k_bitcvt_chunk<<<grid_for(nchunks, 1, smc, 8), 256, 0, st>>>(G, nchunks, cs);
        return check_launch("bit-level chunk");
    };
    gf2x_status s0;
    if (chunked && inverse && (s0 = run_chunks()) != GF2X_OK) return s0;
    struct Group { bool words; std::vector<CvtOp> ops; };
    std::vector<Group> groups;
    for (const CvtOp& op : ops) {
        const bool words = op.lg - 1 - op.K >= 6 && !env_flag("GF2X_BITCVT_SWEEPS");
        if (groups.empty() || groups.back().words != words) groups.push_back({words, {}});
        groups.back().ops.push_back(op);
    }
    if (inverse) std::reverse(groups.begin(), groups.end());
    const uint64_t nw = 1ull << (M - 6);
    InwordSweeps iw;
    iw.n = 0;
    auto flush = [&]() {
        if (!iw.n) return;
        ProfScope ps("k_bitcvt_inword", 16.0 * nw, st);
        k_bitcvt_inword<<<grid_for(nw, 256, smc, 8), 256, 0, st>>>(G, nw, iw);
        iw.n = 0;
    };
    gf2x_status s;
    for (const Group& gr : groups) {
        if (gr.words) {
            flush();
            std::vector<CvtOp> wops;
            for (const CvtOp& op : gr.ops) wops.push_back({op.lg - 6, op.K});
            const std::vector<CvtPass> passes = plan_cvt_ops(wops, M - 6, 8);
            if ((s = run_cvt<uint64_t>(passes, G, M - 6, 1, inverse, smc, st)) != GF2X_OK) return s;
            continue;
        }
        std::vector<CvtOp> seq = gr.ops;
        if (inverse) std::reverse(seq.begin(), seq.end());
        for (const CvtOp& op : seq) {
            const uint64_t h = 1ull << (op.lg - 1), u = h >> op.K, d = h - u;
            for (int sw = 0; sw < 2; sw++) {
                const bool first = inverse ? sw == 1 : sw == 0;   // sweep 1 (targets [h, h+u)) or sweep 2 ([u, h))
                const uint64_t tlo = first ? h : u, thi = first ? h + u : h;
                if (op.lg <= 6) {   // segments inside a word: a periodic mask, sources in the same word
                    uint64_t pmask = 0;
                    for (uint64_t seg = 0; seg < 64; seg += 2 * h)
                        for (uint64_t t = tlo; t < thi; t++) pmask |= 1ull << (seg + t);
                    if (iw.n == 64) flush();
                    iw.pmask[iw.n] = pmask;
                    iw.d[iw.n++] = (int)d;
                    continue;
                }
                flush();
                const uint64_t ntw = ((thi + 63) >> 6) - (tlo >> 6), total = (nw >> (op.lg - 6)) * ntw;
                ProfScope ps("k_bitcvt_sweep", 16.0 * (double)total, st);
                k_bitcvt_sweep<<<grid_for(total, 256, smc, 8), 256, 0, st>>>(G, nw, op.lg, d, tlo, thi);
            }
        }
    }
    flush();
    if ((s = check_launch("bit-level BasisCvt")) != GF2X_OK) return s;
    if (chunked && !inverse) return run_chunks();
    return GF2X_OK;
}

// ---------------------------------------------------------------------------------------------
// The multiply through the Frobenius bijection E_(beta_(m+64) + V_m) (App. C; R23), in the
// polynomial basis of GF(2^128) so that Alg. 4's dense-multiplier FFT passes serve (alg4.cuh, with the
// displacement term psi^-1(s_k(alpha)) per layer): every evaluation is psi^-1 of the tower value, which
// the field isomorphism carries through the products.
//   bits of a, b -> bit-level BasisCvt (2^(m+7) coefficients) -> encoding e_i = sum_j g[i + j n] C'_j
//   (C'_j = psi^-1 of the 7-layer columns) -> n-point FFT at alpha -> pointmul -> iFFT ->
//   decoding (the inverse of the 128 x 128 map) -> bit scatter -> bit-level iBasisCvt -> the product bits.
// The kernels here are the plain forms (one thread per element / word); DESIGN.md §11 has what is next.
// ---------------------------------------------------------------------------------------------
// constants of one m: [m] psi^-1(s_k(alpha)), [128] columns C'_j, [128] columns of the inverse map
struct FrobConsts {
    uint4 v[32 + 128 + 128];
};
#define FROB_ALPHA 0
#define FROB_COLS 32
#define FROB_INV 160

__global__ void __launch_bounds__(256) k_frob_encode(const uint64_t* __restrict__ G, int m, const uint4* __restrict__ cols,
                                                     uint4* __restrict__ W) {
    __shared__ uint4 C[128];
    if (threadIdx.x < 128) C[threadIdx.x] = cols[threadIdx.x];
    __syncthreads();
    const uint64_t n = 1ull << m;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 x = make_uint4(0, 0, 0, 0);
        for (int j = 0; j < 128; j++) {
            const uint64_t p = i + ((uint64_t)j << m);
            if ((__ldg(G + (p >> 6)) >> (p & 63)) & 1) x = xor4(x, C[j]);
        }
        W[i] = x;
    }
}
__global__ void __launch_bounds__(256) k_frob_decode(const uint4* __restrict__ E, uint64_t n, const uint4* __restrict__ inv,
                                                     uint4* __restrict__ Dv) {
    __shared__ uint4 C[128];
    if (threadIdx.x < 128) C[threadIdx.x] = inv[threadIdx.x];
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 e = E[i];
        const uint32_t w[4] = {e.x, e.y, e.z, e.w};
        uint4 y = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int l = 0; l < 4; l++)
            for (int b = 0; b < 32; b++)
                if ((w[l] >> b) & 1) y = xor4(y, C[32 * l + b]);
        Dv[i] = y;
    }
}
// G[w] bit b = bit j of Dv[i] for the coefficient position p = 64 w + b = i + j n
__global__ void __launch_bounds__(256) k_frob_scatter(const uint4* __restrict__ Dv, int m, uint64_t* __restrict__ G, uint64_t nw) {
    const uint64_t nmask = (1ull << m) - 1;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t v = 0;
        for (int b = 0; b < 64; b++) {
            const uint64_t p = (w << 6) + b, i = p & nmask;
            const uint32_t j = (uint32_t)(p >> m);
            const uint4 d = Dv[i];
            const uint32_t limb = j < 32 ? d.x : (j < 64 ? d.y : (j < 96 ? d.z : d.w));
            v |= (uint64_t)((limb >> (j & 31)) & 1) << b;
        }
        G[w] = v;
    }
}

// staged forms for n >= 256 (m >= 8): a CTA takes 256 consecutive i, i.e. 4 words of each of the 128 planes
// j (word (i0 / 64 + q) + j n / 64), loaded once into shared memory
__global__ void __launch_bounds__(256) k_frob_encode_tiled(const uint64_t* __restrict__ G, int m, const uint4* __restrict__ cols,
                                                           uint4* __restrict__ W) {
    __shared__ uint4 C[128];
    __shared__ uint64_t P[128][4];
    if (threadIdx.x < 128) C[threadIdx.x] = cols[threadIdx.x];
    const uint64_t n = 1ull << m, wstride = n >> 6;
    for (uint64_t blk = blockIdx.x; blk < (n >> 8); blk += gridDim.x) {
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < 512; t += 256) {
            const uint32_t j = t >> 2, q = t & 3;
            P[j][q] = G[blk * 4 + q + j * wstride];
        }
        __syncthreads();
        const uint32_t q = threadIdx.x >> 6, b = threadIdx.x & 63;
        uint4 x = make_uint4(0, 0, 0, 0);
#pragma unroll 8
        for (int j = 0; j < 128; j++)
            if ((P[j][q] >> b) & 1) x = xor4(x, C[j]);
        W[blk * 256 + threadIdx.x] = x;
    }
}
// a CTA takes 64 consecutive i (one word of every plane j): thread j gathers bit j of the 64 decoded vectors
__global__ void __launch_bounds__(128) k_frob_scatter_tiled(const uint4* __restrict__ Dv, int m, uint64_t* __restrict__ G) {
    __shared__ uint4 D[64];
    const uint64_t n = 1ull << m, wstride = n >> 6;
    const uint32_t j = threadIdx.x, limb = j >> 5, sh = j & 31;
    for (uint64_t blk = blockIdx.x; blk < (n >> 6); blk += gridDim.x) {
        __syncthreads();
        if (threadIdx.x < 64) D[threadIdx.x] = Dv[blk * 64 + threadIdx.x];
        __syncthreads();
        uint64_t v = 0;
#pragma unroll 8
        for (int t = 0; t < 64; t++) {
            const uint4 d = D[t];
            const uint32_t w = limb == 0 ? d.x : (limb == 1 ? d.y : (limb == 2 ? d.z : d.w));
            v |= (uint64_t)((w >> sh) & 1) << t;
        }
        G[blk + j * wstride] = v;
    }
}

static bool gf2_inverse128_host(const gf2x_host::u128* col, gf2x_host::u128* out) {
    using gf2x_host::u128;
    u128 A[128], I[128];
    for (int r = 0; r < 128; r++) {
        u128 v = 0;
        for (int j = 0; j < 128; j++) if ((col[j] >> r) & 1) v |= (u128)1 << j;
        A[r] = v; I[r] = (u128)1 << r;
    }
    for (int c = 0; c < 128; c++) {
        int p = -1;
        for (int r = c; r < 128; r++) if ((A[r] >> c) & 1) { p = r; break; }
        if (p < 0) return false;
        std::swap(A[p], A[c]); std::swap(I[p], I[c]);
        for (int r = 0; r < 128; r++) if (r != c && ((A[r] >> c) & 1)) { A[r] ^= A[c]; I[r] ^= I[c]; }
    }
    for (int j = 0; j < 128; j++) {
        u128 v = 0;
        for (int r = 0; r < 128; r++) if ((I[r] >> j) & 1) v |= (u128)1 << r;
        out[j] = v;
    }
    return true;
}

static gf2x_status get_frob_consts(DeviceState* ds, int m, const uint4** out) {
    using namespace gf2x_host;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = ds->frob.find(m);
    if (it != ds->frob.end()) { *out = it->second; return GF2X_OK; }
    const Isomorphism iso = build_isomorphism();
    auto to_poly = [&](u128 x) { u128 r = 0; for (int i = 0; i < 128; i++) if ((x >> i) & 1) r ^= iso.towerToPoly[i]; return r; };
    auto to4 = [](u128 v) { return make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96)); };
    FrobConsts h;
    memset(&h, 0, sizeof(h));
    const u128 alpha = (u128)1 << (m + 64);
    u128 sk = alpha, s7[7];
    for (int k = 0; k < m + 7; k++) {            // sk = s_k(alpha)
        if (k < m) h.v[FROB_ALPHA + k] = to4(to_poly(sk));
        else s7[k - m] = sk;
        sk = s1(sk);
    }
    u128 colp[128], inv[128];
    for (int j = 0; j < 128; j++) {               // C_j = prod_{bit b of j} s_(m+b)(alpha) (the 7 layers' images)
        u128 c = 1;
        for (int b = 0; b < 7; b++) if ((j >> b) & 1) c = tower_mul(c, s7[b]);
        colp[j] = to_poly(c);
        h.v[FROB_COLS + j] = to4(colp[j]);
    }
    if (!gf2_inverse128_host(colp, inv)) return fail(GF2X_EINVAL, "App. C encoding map is singular");
    for (int j = 0; j < 128; j++) h.v[FROB_INV + j] = to4(inv[j]);
    uint4* d = nullptr;
    if (cudaMalloc(&d, sizeof(FrobConsts)) != cudaSuccess) return fail(GF2X_ENOMEM, "App. C constants");
    if (cudaMemcpy(d, &h, sizeof(FrobConsts), cudaMemcpyHostToDevice) != cudaSuccess) { cudaFree(d); return fail(GF2X_ECUDA, "App. C constants"); }
    ds->frob[m] = d;
    *out = d;
    return GF2X_OK;
}

static int frob_m_of(uint64_t L) { int m = 0; while (((uint64_t)128 << m) < L) m++; return m; }

static gf2x_status run_frob_mul(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                DeviceState* ds, cudaStream_t st) {
    const uint64_t na = (a_bits + 63) / 64, nb = (b_bits + 63) / 64;
    if (a_bits == 0 || b_bits == 0) {
        if (na + nb) CUDA_TRY(cudaMemsetAsync(c, 0, (na + nb) * 8, st));
        return GF2X_OK;
    }
    const int m = frob_m_of(a_bits + b_bits - 1), M = m + 7;
    if (m > 26) return fail(GF2X_ETOOBIG, "App. C multiply: more than 2^26 points");
    const uint64_t n = 1ull << m, nw = 1ull << (M - 6);
    const uint4* K;
    DevTablesA4* TA;
    gf2x_status s;
    if ((s = get_frob_consts(ds, m, &K)) != GF2X_OK) return s;
    if ((s = get_tablesA4(ds, &TA)) != GF2X_OK) return s;
    void* ws = nullptr;
    const size_t bytes = 2 * nw * 8 + 2 * n * 16;
    if ((s = stream_workspace(ds, st, bytes, &ws)) != GF2X_OK) return s;
    uint64_t* Ga = reinterpret_cast<uint64_t*>(ws);
    uint64_t* Gb = Ga + nw;
    uint4* Wa = reinterpret_cast<uint4*>(Gb + nw);
    uint4* Wb = Wa + n;
    const int smc = ds->sm_count;
    auto body = [&]() -> gf2x_status {
        gf2x_status r;
        {
            ProfScope ps("k_prep", 16.0 * nw, st, 0.0, 2);
            k_prep<<<grid_for(nw, 256, smc, 8), 256, 0, st>>>(a, na, a_bits, M - 6, 1, Ga);
            k_prep<<<grid_for(nw, 256, smc, 8), 256, 0, st>>>(b, nb, b_bits, M - 6, 1, Gb);
        }
        if ((r = run_bitcvt(Ga, M, false, smc, st)) != GF2X_OK) return r;
        if ((r = run_bitcvt(Gb, M, false, smc, st)) != GF2X_OK) return r;
        {
            ProfScope ps("k_frob_encode", 2.0 * (16.0 * n + 16.0 * n), st, 0.0, 2);
            if (m >= 8) {
                k_frob_encode_tiled<<<grid_for(n >> 8, 1, smc, 8), 256, 0, st>>>(Ga, m, K + FROB_COLS, Wa);
                k_frob_encode_tiled<<<grid_for(n >> 8, 1, smc, 8), 256, 0, st>>>(Gb, m, K + FROB_COLS, Wb);
            } else {
                k_frob_encode<<<grid_for(n, 256, smc, 8), 256, 0, st>>>(Ga, m, K + FROB_COLS, Wa);
                k_frob_encode<<<grid_for(n, 256, smc, 8), 256, 0, st>>>(Gb, m, K + FROB_COLS, Wb);
            }
        }
        const std::vector<A4Pass> passes = plan_a4(m);
        for (const A4Pass& f : passes)   // Wa | Wb contiguous: both in one launch per pass
            if ((r = launch_a4(f, false, Wa, n, m, 2, TA, smc, st, K + FROB_ALPHA)) != GF2X_OK) return r;
        {
            ProfScope ps("k_a4_pointmul", 48.0 * n, st);
            k_a4_pointmul<<<grid_for(n, 128, smc, 8), 128, 0, st>>>(Wa, Wb, n);
        }
        for (size_t i = passes.size(); i-- > 0;)
            if ((r = launch_a4(passes[i], true, Wa, n, m, 1, TA, smc, st, K + FROB_ALPHA)) != GF2X_OK) return r;
        {
            ProfScope ps("k_frob_decode", 32.0 * n, st);
            k_frob_decode<<<grid_for(n, 256, smc, 8), 256, 0, st>>>(Wa, n, K + FROB_INV, Wb);
        }
        {
            ProfScope ps("k_frob_scatter", 8.0 * nw + 16.0 * n, st);
            if (m >= 6) k_frob_scatter_tiled<<<grid_for(n >> 6, 1, smc, 16), 128, 0, st>>>(Wb, m, Ga);
            else k_frob_scatter<<<grid_for(nw, 256, smc, 8), 256, 0, st>>>(Wb, m, Ga, nw);
        }
        if ((r = run_bitcvt(Ga, M, true, smc, st)) != GF2X_OK) return r;
        const uint64_t ncopy = std::min<uint64_t>(na + nb, nw);
        CUDA_TRY(cudaMemcpyAsync(c, Ga, ncopy * 8, cudaMemcpyDeviceToDevice, st));
        if (na + nb > ncopy) CUDA_TRY(cudaMemsetAsync(c + ncopy, 0, (na + nb - ncopy) * 8, st));
        return check_launch("App. C multiply");
    };
    return body();
}
