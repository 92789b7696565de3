// alg4.cuh -- the paper's Alg. 4 "simple" multiplication (sec 3.1),
// included by gf2x.cu: BasisCvt on 64-bit blocks, then FFT_LCH directly in GF(2^128) = GF(2)[z]/(z^128 +
// z^7 + z^2 + z + 1) (polynomial basis, no changeRepr) at the points psi^-1(phi_v(i)), i.e. with the
// multipliers s_k(phi_v(b)) computed in the Cantor/tower basis and mapped by the field isomorphism
// (P:573-576): dense, "random-looking 128-bit polynomials".  It is the comparison point that measures
// what the tower's small-subfield multipliers buy on B200 (the product path keeps Alg. 5).
//
// Multiplication by a dense constant c':
//   layers >= 6 (a constant serves >= 64 butterflies): M4R-4 table of c' (32 nibble positions x 16
//     entries x 16 B = 8 KB, word-planar), 128 conflict-free LDS.32 per product;
//   layers < 6: a 16-entry table c' n (256 B) and Horner over the 32 nibbles of x (x c' =
//     sum_t (c' nib_t) z^(4t)).
// Multipliers: c'(k, b) = XOR over the set bits j > k of b of D[k][j], D[k][j] = psi^-1(s_k(v_j))
// (GF(2)-linearity of s_k and psi^-1; host table of 32 x 32 dense images).
#pragma once

typedef unsigned __int128 a4u128;

struct DevTablesA4 {
    uint4 D[32 * 32];   // psi^-1(s_k(v_j)), k, j < 32
};

static void host_build_tablesA4(DevTablesA4* T, const DevTables* host) {
    using namespace gf2x_host;
    const Isomorphism iso = build_isomorphism();
    for (int k = 0; k < 32; k++)
        for (int j = 0; j < 32; j++) {
            const uint32_t s = host->S[k * 32 + j];
            u128 v = 0;
            for (int i = 0; i < 32; i++)
                if ((s >> i) & 1) v ^= iso.towerToPoly[i];
            T->D[k * 32 + j] = make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96));
        }
}

__device__ __forceinline__ a4u128 a4_from(uint4 v) {
    return ((a4u128)v.w << 96) | ((a4u128)v.z << 64) | ((a4u128)v.y << 32) | (a4u128)v.x;
}
__device__ __forceinline__ uint4 a4_to(a4u128 x) {
    return make_uint4((uint32_t)x, (uint32_t)(x >> 32), (uint32_t)(x >> 64), (uint32_t)(x >> 96));
}
// x z^s mod (z^128 + z^7 + z^2 + z + 1), 0 <= s < 128
__device__ __forceinline__ a4u128 a4_mulz(a4u128 x, int s) {
    if (s == 0) return x;
    const a4u128 h = x >> (128 - s);                      // coefficients that leave the field (degree < s)
    a4u128 t = h ^ (h << 1) ^ (h << 2) ^ (h << 7);        // h (z^7 + z^2 + z + 1) ...
    const a4u128 o = (h >> 127) ^ (h >> 126) ^ (h >> 121);  // ... whose own overflow (degree < 7)
    t ^= o ^ (o << 1) ^ (o << 2) ^ (o << 7);
    return (x << s) ^ t;
}
// dense multiplier of layer k, block base b
__device__ __forceinline__ a4u128 a4_const(const uint4* __restrict__ D, int k, uint32_t b) {
    a4u128 c = 0;
    b >>= (k + 1);
    for (int j = k + 1; b; j++, b >>= 1)
        if (b & 1) c ^= a4_from(D[k * 32 + j]);
    return c;
}
// x z^4 mod the field polynomial on 32-bit words (the top nibble folds back as o (z^7 + z^2 + z + 1))
__device__ __forceinline__ uint4 a4_mulz4(uint4 a) {
    const uint32_t o = a.w >> 28;
    uint4 r;
    r.w = __funnelshift_l(a.z, a.w, 4);
    r.z = __funnelshift_l(a.y, a.z, 4);
    r.y = __funnelshift_l(a.x, a.y, 4);
    r.x = (a.x << 4) ^ o ^ (o << 1) ^ (o << 2) ^ (o << 7);
    return r;
}
// x c' by Horner over the 32 nibbles of x (top first) with H[n] = c' n
__device__ __forceinline__ uint4 a4_horner(const uint4* H, uint4 x) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int L = 3; L >= 0; L--)
#pragma unroll
        for (int n = 7; n >= 0; n--) acc = xor4(a4_mulz4(acc), H[(w[L] >> (4 * n)) & 15]);
    return acc;
}
// x c' with the M4R-4 table of c', stored word-planar: T32[w][t][n] = word w of c' n z^(4t) (4 x 2 KB), so
// every lookup is a conflict-free 32-bit load (16 entries of a row sit in 16 distinct banks; 16-byte
// entries put 2 of the 16 candidates in each bank group and conflict)
__device__ __forceinline__ uint4 a4_m4r(const uint4* T, uint4 x) {
    const uint32_t* T32 = reinterpret_cast<const uint32_t*>(T);
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int L = 0; L < 4; L++)
#pragma unroll
        for (int n = 0; n < 8; n++) {
            const uint32_t e = (L * 8 + n) * 16 + ((w[L] >> (4 * n)) & 15);
            acc.x ^= T32[e]; acc.y ^= T32[512 + e]; acc.z ^= T32[1024 + e]; acc.w ^= T32[1536 + e];
        }
    return acc;
}

struct A4Params {
    const uint4* src;
    uint4* dst;
    const uint4* D;
    const uint4* alpha;   // null, or per layer k the displacement term psi^-1(s_k(alpha)) (App. C, frob.cuh)
    uint64_t N, batch;
    int m, c, k_lo, k_hi;
};

// One pass of layers [k_lo, k_hi) on tiles [0,c) U [k_lo,k_hi) (as k_fft2), R = k_hi - k_lo.
// DENSE: M4R-4 tables (R <= 3, 8 KB per multiplier); else Horner tables (R <= 6, 256 B per multiplier).
#define A4_THREADS 256
template <bool INV, bool DENSE>
__global__ void __launch_bounds__(A4_THREADS) k_fft_a4(A4Params p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int R = p.k_hi - p.k_lo;
    const uint32_t nslots = 1u << (p.c + R), ntab = (1u << R) - 1;
    const uint32_t tab_words = DENSE ? 512 : 16;   // uint4 per table
    uint4* tabs = reinterpret_cast<uint4*>(smem_raw);
    uint4* cz = tabs + ntab * tab_words;   // [ntab][4]: c' z^i
    uint4* tile = cz + ntab * 4;
    const uint64_t N = p.N, tiles_per_pair = N >> (p.c + R), ntiles = tiles_per_pair * p.batch;
    const uint32_t cmask = (1u << p.c) - 1;
    const int midbits = p.k_lo - p.c;
    const uint64_t per_cta = ntiles / gridDim.x, extra = ntiles % gridDim.x;
    const uint64_t t_begin = blockIdx.x * per_cta + min((uint64_t)blockIdx.x, extra);
    const uint64_t t_end = t_begin + per_cta + (blockIdx.x < extra ? 1 : 0);
    uint32_t tab_key = 0xFFFFFFFFu;
    for (uint64_t t = t_begin; t < t_end; t++) {
        const uint64_t pair = t / tiles_per_pair;
        const uint32_t tt = (uint32_t)(t - pair * tiles_per_pair);
        const uint32_t base = ((tt & ((1u << midbits) - 1)) << p.c) | ((uint32_t)((uint64_t)(tt >> midbits) << p.k_hi));
        __syncthreads();   // previous tile stored, tables free
        const uint32_t key = (uint32_t)((uint64_t)base >> p.k_hi);
        if (key != tab_key) {   // multipliers depend on the index bits above each layer only
            // (a) one thread per multiplier: c' and its multiples c' z^i, i < 4
            for (uint32_t id = threadIdx.x; id < ntab; id += blockDim.x) {
                const int lg = 31 - __clz(id + 1);
                const int k = p.k_lo + R - 1 - lg;
                const uint32_t blk = id + 1 - (1u << lg);
                const uint32_t lb = (uint32_t)(((uint64_t)base & ~((2ull << k) - 1)) | ((uint64_t)blk << (k + 1)));
                a4u128 cc = a4_const(p.D, k, lb);
                if (p.alpha) cc ^= a4_from(p.alpha[k]);   // s_k(alpha + phi(b)) = s_k(alpha) + s_k(phi(b))
#pragma unroll
                for (int i = 0; i < 4; i++) { cz[id * 4 + i] = a4_to(cc); cc = a4_mulz(cc, 1); }
            }
            __syncthreads();
            // (b) the table entries
            const uint32_t items = ntab * (DENSE ? 32 : 16);
            for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
                const uint32_t id = it / (DENSE ? 32 : 16), sub = it % (DENSE ? 32 : 16);
                uint4* T = tabs + id * tab_words;
                if (DENSE) {   // row sub: entries c' n z^(4 sub)
                    uint4 bz[4];
#pragma unroll
                    for (int i = 0; i < 4; i++) bz[i] = a4_to(a4_mulz(a4_from(cz[id * 4 + i]), 4 * sub));
                    uint32_t* T32 = reinterpret_cast<uint32_t*>(T);
#pragma unroll
                    for (int n = 0; n < 16; n++) {
                        uint4 v = make_uint4(0, 0, 0, 0);
#pragma unroll
                        for (int i = 0; i < 4; i++) if ((n >> i) & 1) v = xor4(v, bz[i]);
                        const uint32_t e = sub * 16 + n;
                        T32[e] = v.x; T32[512 + e] = v.y; T32[1024 + e] = v.z; T32[1536 + e] = v.w;
                    }
                } else {       // entry sub: c' sub
                    uint4 v = make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int i = 0; i < 4; i++) if ((sub >> i) & 1) v = xor4(v, cz[id * 4 + i]);
                    T[sub] = v;
                }
            }
            tab_key = key;
        }
        const uint4* src = p.src + pair * N;
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x) tile[s] = src[base | (s & cmask) | ((s >> p.c) << p.k_lo)];
        __syncthreads();
        for (int li = 0; li < R; li++) {
            const int kr = INV ? li : R - 1 - li;   // layer k_lo + kr
            const int lg = R - 1 - kr;
            for (uint32_t q = threadIdx.x; q < nslots / 2; q += blockDim.x) {
                // pair q: insert a 0 at slot bit (c + kr)
                const int sb = p.c + kr;
                const uint32_t s0 = (q & ((1u << sb) - 1)) | ((q >> sb) << (sb + 1)), s1 = s0 | (1u << sb);
                const uint32_t blk = (s0 >> p.c) >> (kr + 1);
                const uint4* T = tabs + ((1u << lg) - 1 + blk) * tab_words;
                uint4 x0 = tile[s0], x1 = tile[s1];
                if (!INV) {
                    x0 = xor4(x0, DENSE ? a4_m4r(T, x1) : a4_horner(T, x1));
                    x1 = xor4(x1, x0);
                } else {
                    x1 = xor4(x1, x0);
                    x0 = xor4(x0, DENSE ? a4_m4r(T, x1) : a4_horner(T, x1));
                }
                tile[s0] = x0;
                tile[s1] = x1;
            }
            __syncthreads();
        }
        uint4* dst = p.dst + pair * N;
        for (uint32_t s = threadIdx.x; s < nslots; s += blockDim.x) dst[base | (s & cmask) | ((s >> p.c) << p.k_lo)] = tile[s];
    }
}

// operand blocks -> GF(2^128) elements: W[o][p][i] = (S[o][p][i], 0) for i < s_per, 0 beyond
__global__ void k_a4_expand(const uint64_t* __restrict__ S, uint64_t s_per, uint64_t N, uint64_t count, uint4* __restrict__ W) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count * N; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = e / N, i = e - p * N;
        const uint64_t w = i < s_per ? S[p * s_per + i] : 0ull;
        W[e] = make_uint4((uint32_t)w, (uint32_t)(w >> 32), 0u, 0u);
    }
}

// pointmul in GF(2^128): A[i] = A[i] B[i] (Horner with a per-thread 16-entry table of B[i] n)
__global__ void __launch_bounds__(128) k_a4_pointmul(uint4* __restrict__ A, const uint4* __restrict__ B, uint64_t n) {
    __shared__ uint4 H[128 * 16];
    uint4* h = H + threadIdx.x * 16;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const a4u128 y = a4_from(B[i]);
        const a4u128 y1 = a4_mulz(y, 1), y2 = a4_mulz(y, 2), y3 = a4_mulz(y, 3);
#pragma unroll
        for (int e = 0; e < 16; e++) {
            a4u128 v = 0;
            if (e & 1) v ^= y;
            if (e & 2) v ^= y1;
            if (e & 4) v ^= y2;
            if (e & 8) v ^= y3;
            h[e] = a4_to(v);
        }
        A[i] = a4_horner(h, A[i]);
    }
}

// InterleavedCombine of the polynomial-basis C_i (no changeRepr):
// out[w] = lo64(C_w) ^ hi64(C_(w-1)), w < n_out, per product (C_i = 0 for i >= N)
__global__ void k_a4_combine(const uint4* __restrict__ C, uint64_t N, uint64_t n_out, uint64_t batch, uint64_t* __restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_out * batch; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = e / n_out, w = e - p * n_out;
        const uint4* cp = C + p * N;
        uint64_t v = 0;
        if (w < N) { const uint4 x = cp[w]; v ^= ((uint64_t)x.y << 32) | x.x; }
        if (w >= 1 && w - 1 < N) { const uint4 x = cp[w - 1]; v ^= ((uint64_t)x.w << 32) | x.z; }
        out[e] = v;
    }
}

// ------------------------------------------------------------------------------ host
static gf2x_status get_tablesA4(DeviceState* ds, DevTablesA4** out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!ds->tabsA4) {
        DevTablesA4* h = new DevTablesA4;
        host_build_tablesA4(h, ds->host);
        DevTablesA4* d = nullptr;
        cudaError_t e = cudaMalloc(&d, sizeof(DevTablesA4));
        if (e != cudaSuccess) { delete h; return fail(GF2X_ENOMEM, "table allocation failed"); }
        e = cudaMemcpy(d, h, sizeof(DevTablesA4), cudaMemcpyHostToDevice);
        delete h;
        if (e != cudaSuccess) { cudaFree(d); return fail(GF2X_ECUDA, cudaGetErrorString(e)); }
        CUDA_TRY(cudaFuncSetAttribute(k_fft_a4<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft_a4<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft_a4<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_fft_a4<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        ds->tabsA4 = d;
    }
    *out = ds->tabsA4;
    return GF2X_OK;
}

struct A4Pass { int c, k_lo, k_hi; bool dense; };
// layers < 6: Horner passes of <= 6 layers; above: M4R-4 passes of <= 3 layers (7 x 8 KB tables)
static std::vector<A4Pass> plan_a4(int m) {
    std::vector<A4Pass> v;   // forward order (top-down)
    int top = m;
    while (top > 6) {
        const int lo = std::max(6, top - 3);
        v.push_back({std::min(5, lo), lo, top, true});
        top = lo;
    }
    if (top > 0) v.push_back({0, 0, top, false});
    return v;
}

static gf2x_status launch_a4(const A4Pass& f, bool inv, uint4* W, uint64_t N, int m, uint64_t batch, const DevTablesA4* T,
                             int smc, cudaStream_t st, const uint4* alpha = nullptr) {
    A4Params prm;
    prm.src = W; prm.dst = W; prm.D = T->D; prm.alpha = alpha;
    prm.N = N; prm.batch = batch; prm.m = m; prm.c = f.c; prm.k_lo = f.k_lo; prm.k_hi = f.k_hi;
    const int R = f.k_hi - f.k_lo;
    const size_t sm = (((size_t)1 << R) - 1) * ((f.dense ? 512 : 16) + 4) * 16 + ((size_t)1 << (f.c + R)) * 16;
    const uint64_t ntiles = (N >> (f.c + R)) * batch;
    const int occ = std::max(1, std::min(4, (int)(200 * 1024 / (sm + 1024))));
    const int threads = (int)std::min<uint64_t>(A4_THREADS, std::max<uint64_t>(32, ((uint64_t)1 << (f.c + R)) / 2));
    const int occ2 = std::max(1, std::min(16, (int)(200 * 1024 / (sm + 1024))));
    const int grid = grid_for(ntiles, 1, smc, threads < A4_THREADS ? occ2 : occ);
    const double bfly = (double)batch * (double)(N / 2) * R;
    ProfScope ps(f.dense ? "k_fft_a4<m4r>" : "k_fft_a4<horner>", (double)batch * N * 32, st, bfly * (f.dense ? 160.0 : 700.0));
    if (inv) { if (f.dense) k_fft_a4<true, true><<<grid, threads, sm, st>>>(prm); else k_fft_a4<true, false><<<grid, threads, sm, st>>>(prm); }
    else { if (f.dense) k_fft_a4<false, true><<<grid, threads, sm, st>>>(prm); else k_fft_a4<false, false><<<grid, threads, sm, st>>>(prm); }
    return check_launch("fft_a4");
}

// stop_stage: 0 = product; 2 = after FFT_LCH (operand a in Wa), 3 = after pointmul
static gf2x_status run_pipeline_a4(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                   const Plan& P, void* ws, DeviceState* ds, cudaStream_t st, int stop_stage) {
    DevTablesA4* TA;
    gf2x_status s = get_tablesA4(ds, &TA);
    if (s != GF2X_OK) return s;
    unsigned char* base = reinterpret_cast<unsigned char*>(ws);
    uint64_t* Sa = reinterpret_cast<uint64_t*>(base + P.off_sa);
    uint64_t* Sb = reinterpret_cast<uint64_t*>(base + P.off_sb);
    uint4* Wa = reinterpret_cast<uint4*>(base + P.off_wa);
    uint4* Wb = reinterpret_cast<uint4*>(base + P.off_wb);
    const int smc = ds->sm_count;
    const uint64_t B = P.batch;
    {
        ProfScope ps("k_prep", (double)B * (P.na + (1ull << P.ma)) * 8, st);
        k_prep<<<grid_for((1ull << P.ma) * B, 256, smc, 8), 256, 0, st>>>(a, P.na, a_bits, P.ma, B, Sa);
    }
    {
        ProfScope ps("k_prep", (double)B * (P.nb + (1ull << P.mb)) * 8, st);
        k_prep<<<grid_for((1ull << P.mb) * B, 256, smc, 8), 256, 0, st>>>(b, P.nb, b_bits, P.mb, B, Sb);
    }
    const bool same = (P.ma == P.mb) && P.off_sb == P.off_sa + (1ull << P.ma) * B * 8;
    if (same) {
        if ((s = run_cvt<uint64_t>(P.cvt_a, Sa, P.ma, 2 * B, false, smc, st)) != GF2X_OK) return s;
    } else {
        if ((s = run_cvt<uint64_t>(P.cvt_a, Sa, P.ma, B, false, smc, st)) != GF2X_OK) return s;
        if ((s = run_cvt<uint64_t>(P.cvt_b, Sb, P.mb, B, false, smc, st)) != GF2X_OK) return s;
    }
    {
        ProfScope ps("k_a4_expand", 24.0 * P.N * B * 2, st, 0.0, 2);
        k_a4_expand<<<grid_for(P.N * B, 256, smc, 8), 256, 0, st>>>(Sa, 1ull << P.ma, P.N, B, Wa);
        k_a4_expand<<<grid_for(P.N * B, 256, smc, 8), 256, 0, st>>>(Sb, 1ull << P.mb, P.N, B, Wb);
    }
    if ((s = check_launch("a4 expand")) != GF2X_OK) return s;
    const std::vector<A4Pass> passes = plan_a4(P.m);
    for (const A4Pass& f : passes)   // Wa | Wb contiguous: both operands in one launch per pass
        if ((s = launch_a4(f, false, Wa, P.N, P.m, 2 * B, TA, smc, st)) != GF2X_OK) return s;
    if (stop_stage == 2) return GF2X_OK;
    {
        ProfScope ps("k_a4_pointmul", 48.0 * P.N * B, st);
        k_a4_pointmul<<<grid_for(P.N * B, 128, smc, 8), 128, 0, st>>>(Wa, Wb, P.N * B);
    }
    if ((s = check_launch("a4 pointmul")) != GF2X_OK) return s;
    if (stop_stage == 3) return GF2X_OK;
    for (size_t i = passes.size(); i-- > 0;)
        if ((s = launch_a4(passes[i], true, Wa, P.N, P.m, B, TA, smc, st)) != GF2X_OK) return s;
    if ((s = run_cvt<uint4>(P.icvt, Wa, P.m, B, true, smc, st)) != GF2X_OK) return s;
    {
        const uint64_t n_out = P.na + P.nb;
        ProfScope ps("k_a4_combine", 16.0 * P.N * B + 8.0 * n_out * B, st);
        k_a4_combine<<<grid_for(n_out * B, 256, smc, 8), 256, 0, st>>>(Wa, P.N, n_out, B, c);
    }
    return check_launch("a4 combine");
}
