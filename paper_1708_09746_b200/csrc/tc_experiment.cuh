// tc_experiment.cuh -- a measured experiment, not on the product path (VERDICT round 1 item 8 / DESIGN.md §7):
// changeRepr^-1 (§4.3: a fixed 128x128 GF(2) matrix per element) as an int8 tensor-core
// product on sm_100a, tcgen05.mma kind::i8 with the accumulator in TMEM.  Included by gf2x.cu.
//
// A tile of 128 elements is the A operand (M = 128 rows, K = 128: one 0/1 byte per input bit, expanded from the
// 16-byte element), the matrix of psi^-1 the B operand (N = 128 outputs x K = 128, bytes B[o][k] = bit o of
// psi^-1(v_k)), D = A B^T in s32 (128 TMEM columns); bit o of psi^-1(element) is bit 0 of D[e][o] (the sum of
// the ANDs of a GF(2) dot product has the XOR as its parity).  One thread per element expands its row into shared
// memory (canonical K-major layout without swizzle: 8 x 16-byte core matrices), one thread issues the four
// K = 32 MMAs and commits them to an mbarrier, every warp reads its 32 TMEM lanes back (tcgen05.ld 32x32b) and
// packs the parities.  The bit-sliced k_ipsi_bs (generated XOR networks) is the product path's changeRepr^-1.
#pragma once

#define TC_THREADS 128

__device__ __forceinline__ uint64_t tc_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SM100 shared-memory matrix descriptor: start address >> 4 [0,14), leading-dimension byte offset >> 4
    // [16,30), stride-dimension byte offset >> 4 [32,46), version 1 [46,48), base offset 0, layout: no swizzle
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void __launch_bounds__(TC_THREADS, 4) k_ipsi_tc(const uint4* __restrict__ P, uint64_t n,
                                                         const DevTables* tabs, uint4* __restrict__ out,
                                                         uint32_t lbo, uint32_t sbo) {
    __shared__ __align__(1024) unsigned char A[128 * 128];
    __shared__ __align__(1024) unsigned char B[128 * 128];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    // canonical K-major, no swizzle: core matrix (row block rb = r / 8, k block kb = k / 16) at (rb * 8 + kb) * 128
    // bytes, its row r % 8 at + 16 (r % 8), byte k % 16
    auto off = [](uint32_t r, uint32_t k) { return (((r >> 3) * 8 + (k >> 4)) << 7) + ((r & 7) << 4) + (k & 15); };
    // B[o][k] = bit o of psi^-1(v_k): column k of the map, from the M4R-8 table (byte k/8, value 1 << k%8)
    for (uint32_t i = tid; i < 128 * 128; i += TC_THREADS) {
        const uint32_t o = i >> 7, k = i & 127;
        const uint4 col = tabs->ipsi[(k >> 3) * 256 + (1u << (k & 7))];
        const uint32_t w = o < 32 ? col.x : (o < 64 ? col.y : (o < 96 ? col.z : col.w));
        B[off(o, k)] = (unsigned char)((w >> (o & 31)) & 1);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    // instruction descriptor, kind::i8: D s32 (2 << 4), A / B u8, both K-major, N >> 3 at [17,23), M >> 4 at [24,29)
    const uint32_t idesc = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t ntiles = (n + 127) >> 7;
    uint32_t phase = 0;
    uint4 vn = make_uint4(0, 0, 0, 0);
    if (((uint64_t)blockIdx.x << 7) + tid < n) vn = P[((uint64_t)blockIdx.x << 7) + tid];
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, phase ^= 1) {
        // ---- expand my element (row tid) into 0/1 bytes; the next tile's element is loaded under the MMA
        const uint64_t e = (t << 7) + tid, en = ((t + gridDim.x) << 7) + tid;
        const uint4 v = vn;
        vn = en < n ? P[en] : make_uint4(0, 0, 0, 0);
        const uint32_t limb[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int kb = 0; kb < 8; kb++) {   // bytes 16 kb .. 16 kb + 15 = bits 16 kb .. of the element
            const uint32_t x = limb[kb >> 1] >> (16 * (kb & 1));
            uint4 q;
            q.x = ((x & 15) * 0x00204081u) & 0x01010101u;
            q.y = (((x >> 4) & 15) * 0x00204081u) & 0x01010101u;
            q.z = (((x >> 8) & 15) * 0x00204081u) & 0x01010101u;
            q.w = (((x >> 12) & 15) * 0x00204081u) & 0x01010101u;
            *reinterpret_cast<uint4*>(A + off(tid, 16 * kb)) = q;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int ks = 0; ks < 4; ks++) {   // K = 32 bytes per MMA: two core matrices along K
                const uint64_t ad = tc_smem_desc(smem_u32(A) + ks * 256, lbo, sbo);
                const uint64_t bd = tc_smem_desc(smem_u32(B) + ks * 256, lbo, sbo);
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(ks) : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                         : "memory");
        }
        {   // bounded wait: a malformed MMA must fail loudly, not hang the GPU
            uint32_t done = 0, spins = 0;
            while (!done) {
                asm volatile(
                    "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                    : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
                if (++spins > (1u << 24)) __trap();
            }
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // ---- D rows of my warp's 32 lanes: 4 loads of 32 columns, bit 0 of each sum
        uint32_t res[4];
#pragma unroll
        for (int cb = 0; cb < 4; cb++) {
            uint32_t r[32];
            const uint32_t ta = tmem + ((warp * 32) << 16) + cb * 32;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint32_t w = 0;
#pragma unroll
            for (int j = 0; j < 32; j++) w |= (r[j] & 1u) << j;
            res[cb] = w;
        }
        if (e < n) out[e] = make_uint4(res[0], res[1], res[2], res[3]);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();   // A may be rewritten (the MMAs that read it completed before the mbarrier fired)
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------------------------------------
// Warp-shuffle formulation of the innermost forward FFT layers (k = 4 .. 0), a measured experiment (VERDICT
// round 1 item 8 / DESIGN.md §7), against k_bottom's bit-sliced layers (`gf2x_experiment_fft_low`).
// One TGF(2^128) element per lane (index bits [0, 5) = lane), so the layer-k partner is lane ^ 2^k (four
// SHFL per butterfly side).  The multiplier s_k(phi(b)) of the pair's block base b splits by linearity into
// C_hi = s_k(bits >= 5 of b) (warp-uniform: an M4R-4 table per warp and layer, 8 lookups per limb) and
// c_lo = s_k(bits [k+1, 5) of b) < 2^(5-k) (lane-dependent: integer products on bytes, R25), the SURVEY's
// "C_warp + c_lane" split.  Both lanes of a pair form x0 + c x1 (SIMT: the product is issued on both sides).
#define SHFL_THREADS 256
__global__ void __launch_bounds__(SHFL_THREADS) k_fft_low_shfl(uint4* __restrict__ A, uint4* __restrict__ B, uint64_t n) {
    __shared__ __align__(16) uint32_t tabs[SHFL_THREADS / 32][128];   // one M4R-4 table per warp
    __shared__ __align__(16) uint32_t KL[5][32][8];                    // c_lo v_b per layer and lane
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = threadIdx.x; i < 5 * 32; i += blockDim.x) {
        const uint32_t k = i >> 5, l = i & 31;
        uint32_t K[8];
        sm_consts<8>(layer_const((int)k, (l >> (k + 1)) << (k + 1)), K);
#pragma unroll
        for (int b = 0; b < 8; b++) KL[k][l][b] = K[b];
    }
    __syncthreads();
    const uint32_t tab_sa = (uint32_t)__cvta_generic_to_shared(tabs[warp]);
    const uint64_t items = 2 * (n >> 5);
    for (uint64_t it = blockIdx.x * (uint64_t)(SHFL_THREADS / 32) + warp; it < items; it += (uint64_t)gridDim.x * (SHFL_THREADS / 32)) {
        uint4* X = it < (n >> 5) ? A : B;
        const uint64_t i0 = (it % (n >> 5)) << 5;
        uint4 x = X[i0 + lane];
#pragma unroll 1
        for (int k = 4; k >= 0; k--) {
            __syncwarp();
            if (lane < 8) build_tab_row(tabs[warp], layer_const(k, (uint32_t)i0), (int)lane, nullptr);
            __syncwarp();
            const uint32_t m = 1u << k;
            const bool low = !(lane & m);
            uint4 y;
            y.x = __shfl_xor_sync(0xffffffffu, x.x, m); y.y = __shfl_xor_sync(0xffffffffu, x.y, m);
            y.z = __shfl_xor_sync(0xffffffffu, x.z, m); y.w = __shfl_xor_sync(0xffffffffu, x.w, m);
            const uint4 x1 = low ? y : x, x0 = low ? x : y;
            const uint32_t* K = KL[k][lane];
            uint4 x0n;
            x0n.x = x0.x ^ m4r4_word_sa(tab_sa, x1.x) ^ smul<8>(x1.x, K);
            x0n.y = x0.y ^ m4r4_word_sa(tab_sa, x1.y) ^ smul<8>(x1.y, K);
            x0n.z = x0.z ^ m4r4_word_sa(tab_sa, x1.z) ^ smul<8>(x1.z, K);
            x0n.w = x0.w ^ m4r4_word_sa(tab_sa, x1.w) ^ smul<8>(x1.w, K);
            x = low ? x0n : make_uint4(x1.x ^ x0n.x, x1.y ^ x0n.y, x1.z ^ x0n.z, x1.w ^ x0n.w);
        }
        X[i0 + lane] = x;
    }
}
