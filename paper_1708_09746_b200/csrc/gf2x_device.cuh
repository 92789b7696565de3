// gf2x_device.cuh -- device building blocks for the sm_100a GF(2)[x] multiplier.
//
// Tower elements TGF(2^128) are uint4 (four 32-bit limbs; limb L holds coordinates 32L..32L+31,
// i.e. limb L is the TGF(2^32) coefficient of v_(32L)).
// FFT multipliers are < 2^32 (they lie in TGF(2^32) for N <= 2^32 points), so by
// Prop. 2 a butterfly multiplies each limb independently by the same TGF(2^32) constant.
#pragma once
#include <stdint.h>

#define GF2X_HD __host__ __device__
#define GF2X_INLINE __forceinline__

namespace gf2x_dev {

// ---------------------------------------------------------------------------------------------
// SWAR multiplication of every small block of a 32-bit word by a generator (tower relations
// x_1^2 = x_1 + 1, x_2^2 = x_2 + x_1).
// ---------------------------------------------------------------------------------------------
// each GF(4) pair (b0 + b1 x1) -> x1 (b0 + b1 x1) = b1 + (b0 + b1) x1
GF2X_HD GF2X_INLINE uint32_t mulx1(uint32_t u) {
    return ((u >> 1) & 0x55555555u) | ((u ^ (u << 1)) & 0xAAAAAAAAu);
}
// each GF(16) nibble (n0 + n1 x2) -> x2 (n0 + n1 x2) = x1 n1 + (n0 + n1) x2
GF2X_HD GF2X_INLINE uint32_t mulx2(uint32_t u) {
    return mulx1((u >> 2) & 0x33333333u) | ((u ^ (u << 2)) & 0xCCCCCCCCu);
}

// each byte (m0 + m1 x3) -> x3 (m0 + m1 x3) = m1 x1x2 + (m0 + m1) x3   (x3^2 = x3 + x1 x2)
GF2X_HD GF2X_INLINE uint32_t mulx3(uint32_t u) {
    return mulx1(mulx2((u >> 4) & 0x0F0F0F0Fu)) | ((u ^ (u << 4)) & 0xF0F0F0F0u);
}
// each 16-bit half (w0 + w1 x4) -> w1 x1x2x3 + (w0 + w1) x4   (x4^2 = x4 + x1 x2 x3)
GF2X_HD GF2X_INLINE uint32_t mulx4(uint32_t u) {
    return mulx1(mulx2(mulx3((u >> 8) & 0x00FF00FFu))) | ((u ^ (u << 8)) & 0xFF00FF00u);
}
// a TGF(2^32) element (h0 + h1 x5) -> h1 x1x2x3x4 + (h0 + h1) x5   (x5^2 = x5 + x1 x2 x3 x4)
GF2X_HD GF2X_INLINE uint32_t mulx5(uint32_t u) {
    return mulx1(mulx2(mulx3(mulx4(u >> 16)))) | ((u ^ (u << 16)) & 0xFFFF0000u);
}
// c v_(4t), t < 8: v_4 = x3, v_8 = x4, v_16 = x5 (the basis v_k = prod of x_(j+1) over the bits j of k)
GF2X_HD GF2X_INLINE uint32_t mul_v4t(uint32_t c, int t) {
    if (t & 1) c = mulx3(c);
    if (t & 2) c = mulx4(c);
    if (t & 4) c = mulx5(c);
    return c;
}

// ---------------------------------------------------------------------------------------------
// Method of four Russians with 4-bit chunks (§4.3-4.4 use M4R; chunk width chosen for sm_100a:
// a 16-entry table row spans 16 banks, so the 32 lanes of a warp never conflict).
// Table for constant c: tab[16 t + x] = c * (x v_(4t)) = (c v_(4t)) * x, x in GF(16), t < 8.
// ---------------------------------------------------------------------------------------------
struct WtTables {  // M4R-8 tables of the fixed linear maps c -> c * v_(4t), t = 1..7
    const uint32_t* wt;  // [7][4][256]
};

// Cooperative build by the 32 lanes of a warp (c warp-uniform).  Lane l writes entries
// 16 (l/4) + 4 (l%4) + {0,1,2,3}.  Caller must __syncwarp() before use.
__device__ GF2X_INLINE void build_tab(uint32_t* tab, uint32_t c, const uint32_t* __restrict__ wt) {
    const int lane = threadIdx.x & 31;
    const int t = lane >> 2, q = lane & 3;
    uint32_t w = c;
    if (t) {
        const uint32_t* T = wt + (t - 1) * 1024;
        w = __ldg(T + (c & 255)) ^ __ldg(T + 256 + ((c >> 8) & 255)) ^
            __ldg(T + 512 + ((c >> 16) & 255)) ^ __ldg(T + 768 + (c >> 24));
    }
    const uint32_t w1 = mulx1(w), w2 = mulx2(w), w3 = mulx1(w2);
    const uint32_t base = ((q & 1) ? w2 : 0u) ^ ((q & 2) ? w3 : 0u);
    uint32_t* d = tab + 16 * t + 4 * q;
    d[0] = base;
    d[1] = base ^ w;
    d[2] = base ^ w1;
    d[3] = base ^ w ^ w1;
}

__device__ GF2X_INLINE uint32_t m4r4_word(const uint32_t* tab, uint32_t x) {
    uint32_t r = tab[x & 15];
    r ^= tab[16 + ((x >> 4) & 15)];
    r ^= tab[32 + ((x >> 8) & 15)];
    r ^= tab[48 + ((x >> 12) & 15)];
    r ^= tab[64 + ((x >> 16) & 15)];
    r ^= tab[80 + ((x >> 20) & 15)];
    r ^= tab[96 + ((x >> 24) & 15)];
    r ^= tab[112 + (x >> 28)];
    return r;
}

__device__ GF2X_INLINE uint4 m4r4_mul(const uint32_t* tab, uint4 a) {
    return make_uint4(m4r4_word(tab, a.x), m4r4_word(tab, a.y), m4r4_word(tab, a.z), m4r4_word(tab, a.w));
}

__device__ GF2X_INLINE uint4 xor4(uint4 a, uint4 b) {
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}

// ---------------------------------------------------------------------------------------------
// 32x32 bit transpose: on return x[j] bit e = (old x[e]) bit j.
// ---------------------------------------------------------------------------------------------
GF2X_HD GF2X_INLINE void transpose32(uint32_t* x) {
    // 32x32 bit transpose in place: bit j of x[k] <-> bit k of x[j].  Stage s swaps the s-bit blocks
    // (x[k] bits [s,2s) of each 2s-block) <-> (x[k+s] bits [0,s)).  The 16- and 8-bit stages are byte
    // permutes (PRMT, 2 per pair); the 4/2/1-bit stages are a shift + 3-input select per word (4 per pair).
#ifdef __CUDA_ARCH__
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const uint32_t a = x[k], b = x[k + 16];
        x[k] = __byte_perm(a, b, 0x5410);
        x[k + 16] = __byte_perm(a, b, 0x7632);
    }
#pragma unroll
    for (int k = 0; k < 32; k = (k + 9) & ~8) {
        const uint32_t a = x[k], b = x[k + 8];
        x[k] = __byte_perm(a, b, 0x6240);
        x[k + 8] = __byte_perm(a, b, 0x7351);
    }
    uint32_t m = 0x0F0F0F0Fu;
#pragma unroll
    for (int s = 4; s > 0; s >>= 1, m ^= (m << s)) {
#pragma unroll
        for (int k = 0; k < 32; k = (k + s + 1) & ~s) {
            const uint32_t a = x[k], b = x[k + s];
            x[k] = (a & m) | ((b << s) & ~m);
            x[k + s] = ((a >> s) & m) | (b & ~m);
        }
    }
#else
    uint32_t m = 0x0000FFFFu;
    for (int s = 16; s > 0; s >>= 1, m ^= (m << s)) {
        for (int k = 0; k < 32; k = (k + s + 1) & ~s) {
            const uint32_t t = ((x[k] >> s) ^ x[k + s]) & m;
            x[k] ^= t << s;
            x[k + s] ^= t;
        }
    }
#endif
}


__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------------------------------------
// TMA (cp.async.bulk[.tensor]) loads completing on an mbarrier with a transaction count (k_cvt_rb_tma)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
// generic-proxy accesses of shared memory ordered before later async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

// bulk prefetch of a global range into L2 (no completion mechanism; a hint)
__device__ __forceinline__ void bulk_prefetch_l2(const void* g, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}
// TMA stores (shared -> global, bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* tmap, int c0, int c1, int c2, int c3, const void* ssrc) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tmap), "r"(c0),
                 "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(ssrc))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }

// cp.async (LDGSTS): 16-byte global -> shared copies that complete asynchronously (no register
// staging), grouped per thread; used to prefetch the next tile while the current one is processed.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace gf2x_dev
