// trunc.cuh -- truncated FFT for products just above a power of two (§5.1: "one can
// truncate the FFT to make the curve somewhat smoother").  Included by gf2x.cu.
//
// The paper gives no truncation algorithm; this one follows from Alg. 1 itself (R21).  With
// N = 2^m points, H = N/2 and a product of L <= H + 2^j novel-basis coefficients g = (g_lo, g_hi), |g_hi| <= 2^j:
//   * the lower half of FFT_N at phi(i), i < H, is FFT_H of the lower half of the coefficients (the top
//     layer's block-0 multiplier is s_(m-1)(0) = 0), and iFFT_H of it returns g_lo exactly (X_k, k >= H,
//     carries the factor s_(m-1), which vanishes on V_(m-1));
//   * on the upper half (alpha + phi(i), alpha = v_(m-1), s_(m-1)(alpha) = 1) the product evaluates
//     h = g_lo + g_hi; its first 2^j values only need the block-0 chain of the upper sub-transform:
//     Reduce(h) = for k = m-2 .. j: h[0, 2^k) += s_k(alpha) h[2^k, 2^(k+1)) (O(H) work), then FFT_j with
//     the multipliers of the global indices H + i;
//   * Reduce is linear and leaves g_hi (support < 2^j) alone, so g_hi = iFFT_j(values) + Reduce(g_lo)[0, 2^j).
// Operands with n_a, n_b <= H have h = (their coefficients), so the forward side is FFT_H + Reduce + FFT_j.
// A multiply of L = H + 1 blocks then costs about one H-point multiply instead of an N-point one.
#pragma once

// x[i] ^= c (x) x[half + i], i < half: one block-0 layer of Reduce (c < 2^32, limb-wise M4R-4), on one
// array or on two (x2 != nullptr: both operands in one launch)
__global__ void __launch_bounds__(256) k_trunc_fold(uint4* __restrict__ x, uint4* __restrict__ x2, uint64_t half,
                                                    uint32_t c, const DevTables* __restrict__ tabs) {
    __shared__ __align__(1024) uint32_t tab[128];
    if (threadIdx.x < 8) build_tab_row(tab + 0, c, threadIdx.x, tabs->wt);
    __syncthreads();
    const uint32_t ta = (uint32_t)__cvta_generic_to_shared(tab);
    const uint64_t total = x2 ? 2 * half : half;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        uint4* y = e < half ? x : x2;
        const uint64_t i = e < half ? e : e - half;
        const uint4 v = y[half + i];
        uint4 a = y[i];
        a.x ^= m4r4_word_sa(ta, v.x); a.y ^= m4r4_word_sa(ta, v.y);
        a.z ^= m4r4_word_sa(ta, v.z); a.w ^= m4r4_word_sa(ta, v.w);
        y[i] = a;
    }
}

// changeRepr of the novel-basis blocks into a scratch of H tower elements: x[i] = psi(S[i]) (i < s_per), 0
// beyond (M4R-8, the same table as the changeRepr FFT pass)
__global__ void __launch_bounds__(256) k_psi64(const uint64_t* __restrict__ S, uint64_t s_per, uint64_t H,
                                               const DevTables* __restrict__ tabs, uint4* __restrict__ x) {
    __shared__ uint4 psit[8 * 256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) psit[i] = tabs->psi64[i];
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < H; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = i < s_per ? S[i] : 0ull;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (w) {
#pragma unroll
            for (int ch = 0; ch < 8; ch++) v = xor4(v, psit[ch * 256 + ((w >> (8 * ch)) & 255)]);
        }
        x[i] = v;
    }
}

// NL layers of Reduce in one pass: layer l (k = k_top - l) folds x[2^k, 2^(k+1)) into x[0, 2^k) times c_l.
// Thread i < Q = 2^(k_top - NL + 1) holds x[i + u Q], u < 2^NL, in registers and folds them down to u = 0.
// PSI: the source is the operand's novel-basis blocks S (s_per words, 0 beyond), changeRepr'ed on the fly;
// else the source is tower elements.  Two operands per launch when src2 != nullptr.  In place is safe
// (thread i writes x[i] and only reads it or elements at or above Q).
struct ReduceArgs {
    const void* src[2];
    uint4* dst[2];
    uint64_t s_per[2];
    uint32_t c[5];
};
template <int NL, bool PSI>
__global__ void __launch_bounds__(256) k_trunc_reduce(ReduceArgs ra, int nops, uint64_t Q, const DevTables* __restrict__ tabs) {
    __shared__ __align__(1024) uint32_t tab[NL * 128];
    __shared__ uint4 psit[PSI ? 8 * 256 : 1];
    if (threadIdx.x < 8 * NL) {
        const int l = threadIdx.x >> 3;
        uint32_t c = ra.c[0];
#pragma unroll
        for (int q = 1; q < NL; q++) c = l == q ? ra.c[q] : c;
        build_tab_row(tab + 128 * l, c, threadIdx.x & 7, tabs->wt);
    }
    if (PSI)
        for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) psit[i] = tabs->psi64[i];
    __syncthreads();
    const uint32_t ta = (uint32_t)__cvta_generic_to_shared(tab);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nops * Q; e += (uint64_t)gridDim.x * blockDim.x) {
        const int op = e >= Q;
        const uint64_t i = e - (op ? Q : 0);
        const void* src = op ? ra.src[1] : ra.src[0];
        const uint64_t s_per = op ? ra.s_per[1] : ra.s_per[0];
        uint4 x[1 << NL];
#pragma unroll
        for (int u = 0; u < (1 << NL); u++) {
            const uint64_t idx = i + (uint64_t)u * Q;
            if (PSI) {
                const uint64_t w = idx < s_per ? reinterpret_cast<const uint64_t*>(src)[idx] : 0ull;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (w) {
#pragma unroll
                    for (int ch = 0; ch < 8; ch++) v = xor4(v, psit[ch * 256 + ((w >> (8 * ch)) & 255)]);
                }
                x[u] = v;
            } else {
                x[u] = reinterpret_cast<const uint4*>(src)[idx];
            }
        }
        if constexpr (NL >= 5) reduce_level<16>(x, ta + 512 * (NL - 5));
        if constexpr (NL >= 4) reduce_level<8>(x, ta + 512 * (NL - 4));
        if constexpr (NL >= 3) reduce_level<4>(x, ta + 512 * (NL - 3));
        if constexpr (NL >= 2) reduce_level<2>(x, ta + 512 * (NL - 2));
        reduce_level<1>(x, ta + 512 * (NL - 1));
        (op ? ra.dst[1] : ra.dst[0])[i] = x[0];
    }
}
template <int NL>
static void launch_trunc_reduce(bool psi, const ReduceArgs& ra, int nops, uint64_t Q, const DevTables* tabs, int smc, cudaStream_t st) {
    const int g = grid_for(nops * Q, 256, smc, 4);
    if (psi) k_trunc_reduce<NL, true><<<g, 256, 0, st>>>(ra, nops, Q, tabs);
    else k_trunc_reduce<NL, false><<<g, 256, 0, st>>>(ra, nops, Q, tabs);
}

// an operand reaching past H: h = a_lo + a_hi on the upper half, and Reduce leaves a_hi (support < 2^j) alone,
// so its changeRepr'ed tail is added to the reduced 2^j elements: U[i] ^= psi(S[H + i]), i < r
__global__ void __launch_bounds__(256) k_trunc_addhi(const uint64_t* __restrict__ S, uint64_t r, const DevTables* __restrict__ tabs,
                                                     uint4* __restrict__ U) {
    __shared__ uint4 psit[8 * 256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) psit[i] = tabs->psi64[i];
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < r; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = S[i];
        uint4 v = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int ch = 0; ch < 8; ch++) v = xor4(v, psit[ch * 256 + ((w >> (8 * ch)) & 255)]);
        U[i] = xor4(U[i], v);
    }
}

struct TruncGeom {
    int m, j;          // N = 2^m points, upper part 2^j
    uint64_t N, H, U;  // U = 2^j
};
// eligible: one product, L - H <= 2^j with 12 <= j <= m - 2 (an operand longer than H has a tail of <= 2^j words)
static bool trunc_geom(const Plan& P, TruncGeom& T) {
    if (env_flag("GF2X_NO_TRUNC") || P.batch != 1 || P.m < 14) return false;
    const uint64_t H = P.N / 2, L = P.na + P.nb - 1;
    if (L <= H) return false;   // (an operand may reach past H: its tail is at most L - H <= 2^j words)
    int j = 12;
    while ((1ull << j) < L - H) j++;
    if (j > P.m - 2) return false;
    T.m = P.m; T.j = j; T.N = P.N; T.H = H; T.U = 1ull << j;
    return true;
}

// the side stream of caller stream st (created on first use; fork / join by events, capturable)
static DeviceState::Aux* get_aux(DeviceState* ds, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceState::Aux& a = ds->aux[st];
    if (!a.s) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&a.s, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming) != cudaSuccess) {
            ds->aux.erase(st);
            return nullptr;
        }
    }
    return &a;
}

// the lower transform's first / last pass folds Reduce's top 6 layers (k_fft2 red_dst) when its geometry fits
static bool trunc_fuse(const std::vector<FftPass>& fl, const TruncGeom& T) {
    return !env_flag("GF2X_TRUNC_LAYERED") && !env_flag("GF2X_TRUNC_NOFUSE") && fl.size() > 1 && fl[0].c == 5 &&
           fl[0].k_hi - fl[0].k_lo == 6 && fl[0].k_hi == T.m - 1 && T.j <= fl[0].k_lo;
}
// R28 on the truncated path (one product): the output words fit N, whole bit-sliced tiles
static bool trunc_mcomb(const Plan& P) {
    return P.na + P.nb <= P.N && P.N % IB_TILE == 0 && !env_flag("GF2X_NO_MCOMB") && !env_flag("GF2X_NO_IPSI_BS");
}
// kernel launches of one truncated multiply (the default variant)
static int launches_of_trunc(const Plan& P, const TruncGeom& T) {
    const std::vector<FftPass> fl = plan_fft(T.m - 1), fu = plan_fft(T.j);
    const bool fuse = trunc_fuse(fl, T);
    const int k0 = fuse ? fl[0].k_lo - 1 : T.m - 2;
    const int nred = k0 >= T.j ? (k0 - T.j + 1 + 4) / 5 : 0;
    int n = 2;                                                             // prep a, b
    n += launches_of_split(P.sa, P.cvt_a, P.ma) + launches_of_split(P.sb, P.cvt_b, P.mb);
    n += 3 * ((int)fl.size() - 1) + 1;                                     // lower: forward a, b, bottom, inverse
    n += 3 * ((int)fu.size() - 1) + 1;                                     // upper
    n += 2 * nred + 1;                                                     // Reduce (forward, g_lo), g_hi combine
    n += (P.na > T.H) + (P.nb > T.H);                                      // operand tails past H
    if (trunc_mcomb(P)) {   // R28: changeRepr^-1 + combine, then the 64-bit iBasisCvt
        const uint64_t n_out = P.na + P.nb;
        n += 1 + launches_of_split(plan_cvt_split(n_out, P.m, 8), P.icvt64, P.m);
    } else {
        n += launches_of_split(P.ic, P.icvt, P.m) + 1;                          // iBasisCvt, changeRepr^-1 + combine
    }
    return n;
}

static gf2x_status run_pipeline_trunc(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                      const Plan& P, const TruncGeom& T, void* ws, DeviceState* ds, cudaStream_t st) {
    unsigned char* base = reinterpret_cast<unsigned char*>(ws);
    uint64_t* Sa = reinterpret_cast<uint64_t*>(base + P.off_sa);
    uint64_t* Sb = reinterpret_cast<uint64_t*>(base + P.off_sb);
    uint4* Wa = reinterpret_cast<uint4*>(base + P.off_wa);
    uint4* Wb = reinterpret_cast<uint4*>(base + P.off_wb);
    const int smc = ds->sm_count;
    const DevTables* H = ds->host;
    gf2x_status s;
    // Split + BasisCvt on the operands (as the full path)
    {
        ProfScope ps("k_prep", (double)(P.na + (1ull << P.ma)) * 8, st);
        k_prep<<<grid_for(1ull << P.ma, 256, smc, 8), 256, 0, st>>>(a, P.na, a_bits, P.ma, 1, Sa);
    }
    {
        ProfScope ps("k_prep", (double)(P.nb + (1ull << P.mb)) * 8, st);
        k_prep<<<grid_for(1ull << P.mb, 256, smc, 8), 256, 0, st>>>(b, P.nb, b_bits, P.mb, 1, Sb);
    }
    if ((s = run_cvt_operand(P, true, Sa, smc, st)) != GF2X_OK) return s;
    if ((s = run_cvt_operand(P, false, Sb, smc, st)) != GF2X_OK) return s;
    // sub-plans: lower part (H points, global index = local) and upper part (2^j points at H + i)
    Plan PL;
    PL.N = T.H; PL.m = T.m - 1; PL.batch = 1;
    const std::vector<FftPass> fl = plan_fft(T.m - 1);
    Plan PU;
    PU.N = T.U; PU.m = T.j; PU.batch = 1;
    const std::vector<FftPass> fu = plan_fft(T.j);
    const IdxMap umap{T.j, T.m - T.j, (uint32_t)(T.H >> T.j)};
    uint4* Ua = Wa + T.H;   // upper scratch: H elements per operand
    uint4* Ub = Wb + T.H;
    // Reduce(h), k = m-2 .. j, in passes of up to 5 layers (the first one reading src / changeRepr'ing S);
    // the result, 2^j elements per operand, lands in dst[0, 2^j)
    auto reduce = [&](bool psi, ReduceArgs ra, int nops, cudaStream_t st, int k0) -> gf2x_status {
        if (env_flag("GF2X_TRUNC_LAYERED")) {   // debug: one launch per layer, through the H-element scratch
            if (psi) {
                ProfScope ps("k_psi64", (double)nops * T.H * 24, st);
                for (int o = 0; o < nops; o++)
                    k_psi64<<<grid_for(T.H, 256, smc, 8), 256, 0, st>>>((const uint64_t*)ra.src[o], ra.s_per[o], T.H, ds->tabs, ra.dst[o]);
            } else {
                for (int o = 0; o < nops; o++) CUDA_TRY(cudaMemcpyAsync(ra.dst[o], ra.src[o], T.H * 16, cudaMemcpyDeviceToDevice, st));
            }
            for (int k = T.m - 2; k >= T.j; k--) {
                const uint64_t half = 1ull << k;
                ProfScope ps("k_trunc_fold", 48.0 * half * nops, st);
                k_trunc_fold<<<grid_for(half * nops, 256, smc, 8), 256, 0, st>>>(ra.dst[0], nops > 1 ? ra.dst[1] : nullptr, half,
                                                                                 H->S[k * 32 + (T.m - 1)], ds->tabs);
            }
            return check_launch("trunc fold");
        }
        bool first = true;
        for (int k = k0; k >= T.j;) {
            const int nl = std::min(5, k - T.j + 1);
            const uint64_t Q = 1ull << (k - nl + 1);
            for (int l = 0; l < nl; l++) ra.c[l] = H->S[(k - l) * 32 + (T.m - 1)];
            if (!first) { ra.src[0] = ra.dst[0]; ra.src[1] = ra.dst[1]; }
            const bool p = psi && first;
            ProfScope ps("k_trunc_reduce", (double)nops * Q * ((p ? 8.0 : 16.0) * (1 << nl) + 16.0), st);
            switch (nl) {
                case 1: launch_trunc_reduce<1>(p, ra, nops, Q, ds->tabs, smc, st); break;
                case 2: launch_trunc_reduce<2>(p, ra, nops, Q, ds->tabs, smc, st); break;
                case 3: launch_trunc_reduce<3>(p, ra, nops, Q, ds->tabs, smc, st); break;
                case 4: launch_trunc_reduce<4>(p, ra, nops, Q, ds->tabs, smc, st); break;
                default: launch_trunc_reduce<5>(p, ra, nops, Q, ds->tabs, smc, st); break;
            }
            k -= nl;
            first = false;
        }
        return check_launch("trunc reduce");
    };
    // the lower part's first pass (changeRepr + the top 6 layers) also folds its 6 index bits for Reduce
    const bool fuse = trunc_fuse(fl, T);
    auto lower_pass = [&](size_t i) -> gf2x_status {
        const bool first = i == 0;
        uint32_t rc[6];
        if (first && fuse)
            for (int kk = 0; kk < 6; kk++) rc[kk] = H->S[(fl[0].k_lo + kk) * 32 + (T.m - 1)];
        gf2x_status r;
        if ((r = launch_fft(fl[i], false, first, first ? (const void*)Sa : Wa, first ? (1ull << P.ma) : T.H, Wa, PL, ds, st, 1,
                            IdxMap{0, 0, 0}, first && fuse ? Ua : nullptr, rc)) != GF2X_OK)
            return r;
        return launch_fft(fl[i], false, first, first ? (const void*)Sb : Wb, first ? (1ull << P.mb) : T.H, Wb, PL, ds, st, 1,
                          IdxMap{0, 0, 0}, first && fuse ? Ub : nullptr, rc);
    };
    if (fuse && (s = lower_pass(0)) != GF2X_OK) return s;
    // upper part (on the side stream when available: its small, latency-bound launches overlap the lower
    // part's): Reduce of the operands' (changeRepr'ed) coefficients to 2^j, FFT_j at H + i, bottom, iFFT_j
    DeviceState::Aux* aux = env_flag("GF2X_TRUNC_SERIAL") ? nullptr : get_aux(ds, st);
    const cudaStream_t su = aux ? aux->s : st;
    if (aux) {
        CUDA_TRY(cudaEventRecord(aux->fork, st));
        CUDA_TRY(cudaStreamWaitEvent(su, aux->fork, 0));
    }
    // an early error return still joins the side stream back into st (nothing of this call keeps running
    // on the workspace after it returns control of st)
    struct JoinGuard {
        DeviceState::Aux* a; cudaStream_t st, su; bool recorded = false, joined = false;
        ~JoinGuard() {
            if (!a) return;
            if (!recorded) cudaEventRecord(a->join, su);
            if (!joined) cudaStreamWaitEvent(st, a->join, 0);
        }
    } jg{aux, st, su};
    {
        ReduceArgs ra{};
        ra.src[0] = fuse ? (const void*)Ua : Sa; ra.src[1] = fuse ? (const void*)Ub : Sb;
        ra.s_per[0] = 1ull << P.ma; ra.s_per[1] = 1ull << P.mb;
        ra.dst[0] = Ua; ra.dst[1] = Ub;
        if ((s = reduce(!fuse, ra, 2, su, fuse ? fl[0].k_lo - 1 : T.m - 2)) != GF2X_OK) return s;
    }
    for (int o = 0; o < 2; o++) {   // operand tails past H
        const uint64_t n = o ? P.nb : P.na;
        if (n <= T.H) continue;
        ProfScope ps("k_trunc_addhi", (double)(n - T.H) * 40, su);
        k_trunc_addhi<<<grid_for(n - T.H, 256, smc, 4), 256, 0, su>>>((o ? Sb : Sa) + T.H, n - T.H, ds->tabs, o ? Ub : Ua);
    }
    for (size_t i = 0; i + 1 < fu.size(); i++) {
        if ((s = launch_fft(fu[i], false, false, Ua, T.U, Ua, PU, ds, su, 1, umap)) != GF2X_OK) return s;
        if ((s = launch_fft(fu[i], false, false, Ub, T.U, Ub, PU, ds, su, 1, umap)) != GF2X_OK) return s;
    }
    {
        BottomParams bp;
        bp.A = Ua; bp.B = Ub;
        bp.total = T.U;
        bp.ntiles = (T.U + (1ull << BT_BITS) - 1) >> BT_BITS;
        bp.m = T.j; bp.L = fu.back().layers; bp.mode = 7; bp.map = umap;
        ProfScope ps("k_bottom", 48.0 * T.U, su, bottom_alu_ops(bp));
        bottom_launch(bp, smc, su);
    }
    for (size_t i = fu.size() - 1; i-- > 0;)
        if ((s = launch_fft(fu[i], true, false, Ua, T.U, Ua, PU, ds, su, 1, umap)) != GF2X_OK) return s;
    if (aux) { CUDA_TRY(cudaEventRecord(aux->join, su)); jg.recorded = true; }
    // lower part: the H-point multiply of the full pipeline (changeRepr fused into its first pass)
    for (size_t i = fuse ? 1 : 0; i + 1 < fl.size(); i++)
        if ((s = lower_pass(i)) != GF2X_OK) return s;
    if (fl.size() == 1) return fail(GF2X_EINVAL, "truncated path needs a table pass");   // (m - 1 >= 13 always has one)
    {
        BottomParams bp;
        bp.A = Wa; bp.B = Wb;
        bp.total = T.H;
        bp.ntiles = (T.H + (1ull << BT_BITS) - 1) >> BT_BITS;
        bp.m = T.m - 1; bp.L = fl.back().layers; bp.mode = 7; bp.map = IdxMap{0, 0, 0};
        ProfScope ps("k_bottom", 48.0 * T.H, st, bottom_alu_ops(bp));
        bottom_launch(bp, smc, st);
    }
    // g_hi = iFFT_j(...) + Reduce(g_lo)[0, 2^j): Reduce of g_lo (in Wa) into Wb (free now); fused, the last
    // inverse pass folds its top 6 index bits on the way out
    uint32_t rc[6];
    for (int kk = 0; kk < 6 && fuse; kk++) rc[kk] = H->S[(fl[0].k_lo + kk) * 32 + (T.m - 1)];
    for (size_t i = fl.size() - 1; i-- > 0;)
        if ((s = launch_fft(fl[i], true, false, Wa, T.H, Wa, PL, ds, st, 1, IdxMap{0, 0, 0}, fuse && i == 0 ? Wb : nullptr, rc)) != GF2X_OK)
            return s;
    {
        ReduceArgs ra{};
        ra.src[0] = fuse ? (const void*)Wb : Wa;
        ra.dst[0] = Wb;
        if ((s = reduce(false, ra, 1, st, fuse ? fl[0].k_lo - 1 : T.m - 2)) != GF2X_OK) return s;
    }
    if (aux) { CUDA_TRY(cudaStreamWaitEvent(st, aux->join, 0)); jg.joined = true; }
    {
        ProfScope ps("k_xor_range", 48.0 * T.U, st);
        k_xor_range<<<grid_for(T.U, 256, smc, 8), 256, 0, st>>>(Ua - 0, Wb - 0, 0, T.U);
    }
    const uint64_t n_out = P.na + P.nb;
    if ((s = check_launch("trunc combine")) != GF2X_OK) return s;
    if (trunc_mcomb(P)) {
        // R28: changeRepr^-1 and the combine written in the novel basis (the coefficients g_k, k >= H + U, are zero:
        // read as 0, no clearing), then iBasisCvt of the n_out 64-bit words -- split at 2^p + 2^j (R22) as the
        // 128-bit path would be -- in the output when the split's extent fits it, else in Wb (then copied)
        const CvtSplit S64 = plan_cvt_split(n_out, P.m, 8);
        const uint64_t extent = S64.p >= 0 ? (1ull << S64.p) + (1ull << S64.j) : P.N;
        uint64_t* D = (extent <= n_out && ((uintptr_t)c & 15) == 0) ? c : reinterpret_cast<uint64_t*>(Wb);
        if (D != c && extent > n_out) CUDA_TRY(cudaMemsetAsync(D + n_out, 0, (extent - n_out) * 8, st));
        {
            ProfScope ps("k_ipsi_mcomb", 16.0 * n_out + 8.0 * n_out, st);
            k_ipsi_bs<true><<<grid_for((n_out + IB_TILE - 1) / IB_TILE, 1, smc, 2), IB_THREADS, 6 * IB_TILE * 4, st>>>(
                Wa, ds->tabs, P.N, 1, D, nullptr, n_out, T.H + T.U);
        }
        if ((s = check_launch("trunc mcomb")) != GF2X_OK) return s;
        s = S64.p >= 0 ? run_icvt_split<uint64_t>(S64, D, smc, st) : run_cvt<uint64_t>(P.icvt64, D, P.m, 1, true, smc, st);
        if (s != GF2X_OK) return s;
        if (D != c) CUDA_TRY(cudaMemcpyAsync(c, D, n_out * 8, cudaMemcpyDeviceToDevice, st));
        return GF2X_OK;
    }
    // iBasisCvt on the N coefficients (or split at H, R22: only units < n_out are read afterwards), then
    // changeRepr^-1 + InterleavedCombine (as the full path)
    if (P.ic.p >= 0) {
        if (n_out > T.H + T.U) CUDA_TRY(cudaMemsetAsync(Ua + T.U, 0, (n_out - T.H - T.U) * 16, st));
        if ((s = run_icvt_split(P.ic, Wa, smc, st)) != GF2X_OK) return s;
    } else {
        CUDA_TRY(cudaMemsetAsync(Ua + T.U, 0, (T.H - T.U) * 16, st));
        if ((s = run_cvt<uint4>(P.icvt, Wa, P.m, 1, true, smc, st)) != GF2X_OK) return s;
    }
    if (n_out <= P.N && P.N % IB_TILE == 0 && !env_flag("GF2X_NO_IPSI_BS")) {
        ProfScope ps("k_ipsi_bs", 16.0 * n_out + 8.0 * n_out, st);
        k_ipsi_bs<false><<<grid_for((n_out + IB_TILE - 1) / IB_TILE, 1, smc, 2), IB_THREADS, 6 * IB_TILE * 4, st>>>(Wa, ds->tabs, P.N,
                                                                                                        1, c, nullptr, n_out);
    } else {
        ProfScope ps("k_ipsi_combine", 16.0 * P.N + 8.0 * n_out, st);
        k_ipsi_combine<<<grid_for(n_out, 256, smc, 2), 256, 16 * 256 * 16, st>>>(Wa, ds->tabs, P.N, n_out, 1, c, nullptr);
    }
    return check_launch("trunc ipsi");
}

// mul_common's hook: 1 if the product took the truncated path (*out = its status), 0 otherwise
static int run_trunc_if_eligible(const uint64_t* a, uint64_t a_bits, const uint64_t* b, uint64_t b_bits, uint64_t* c,
                                 const Plan& P, void* ws, DeviceState* ds, cudaStream_t st, gf2x_status* out) {
    TruncGeom T;
    if (!trunc_geom(P, T)) return 0;
    *out = run_pipeline_trunc(a, a_bits, b, b_bits, c, P, T, ws, ds, st);
    return 1;
}
