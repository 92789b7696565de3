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

struct TruncGeom {
    int m, j;          // N = 2^m points, upper part 2^j
    uint64_t N, H, U;  // U = 2^j
};
// eligible: one product, both operands within the lower half, L - H <= 2^j with 12 <= j <= m - 2
static bool trunc_geom(const Plan& P, TruncGeom& T) {
    if (env_flag("GF2X_NO_TRUNC") || P.batch != 1 || P.m < 14) return false;
    const uint64_t H = P.N / 2, L = P.na + P.nb - 1;
    if (P.na > H || P.nb > H || L <= H) return false;
    int j = 12;
    while ((1ull << j) < L - H) j++;
    if (j > P.m - 2) return false;
    T.m = P.m; T.j = j; T.N = P.N; T.H = H; T.U = 1ull << j;
    return true;
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
    // upper part, forward: changeRepr of the coefficients into the scratch, Reduce to 2^j, FFT_j at H + i
    {
        ProfScope ps("k_psi64", 2.0 * T.H * 24, st);
        k_psi64<<<grid_for(T.H, 256, smc, 8), 256, 0, st>>>(Sa, 1ull << P.ma, T.H, ds->tabs, Ua);
        k_psi64<<<grid_for(T.H, 256, smc, 8), 256, 0, st>>>(Sb, 1ull << P.mb, T.H, ds->tabs, Ub);
    }
    if ((s = check_launch("trunc psi")) != GF2X_OK) return s;
    auto reduce = [&](uint4* x, uint4* x2) -> gf2x_status {
        for (int k = T.m - 2; k >= T.j; k--) {
            const uint64_t half = 1ull << k;
            ProfScope ps("k_trunc_fold", 48.0 * half * (x2 ? 2 : 1), st);
            k_trunc_fold<<<grid_for(half * (x2 ? 2 : 1), 256, smc, 8), 256, 0, st>>>(x, x2, half, H->S[k * 32 + (T.m - 1)],
                                                                                   ds->tabs);
        }
        return check_launch("trunc fold");
    };
    if ((s = reduce(Ua, Ub)) != GF2X_OK) return s;
    for (size_t i = 0; i + 1 < fu.size(); i++) {
        if ((s = launch_fft(fu[i], false, false, Ua, T.U, Ua, PU, ds, st, 1, umap)) != GF2X_OK) return s;
        if ((s = launch_fft(fu[i], false, false, Ub, T.U, Ub, PU, ds, st, 1, umap)) != GF2X_OK) return s;
    }
    {
        BottomParams bp;
        bp.A = Ua; bp.B = Ub;
        bp.total = T.U;
        bp.ntiles = (T.U + (1ull << BT_BITS) - 1) >> BT_BITS;
        bp.m = T.j; bp.L = fu.back().layers; bp.mode = 7; bp.map = umap;
        ProfScope ps("k_bottom", 48.0 * T.U, st, (double)bp.ntiles * (3.0 * bp.L * 128.0 + 576.0) * OPS_BS_MUL32);
        bottom_launch(bp, smc, st);
    }
    for (size_t i = fu.size() - 1; i-- > 0;)
        if ((s = launch_fft(fu[i], true, false, Ua, T.U, Ua, PU, ds, st, 1, umap)) != GF2X_OK) return s;
    // lower part: the H-point multiply of the full pipeline (changeRepr fused into its first pass)
    for (size_t i = 0; i + 1 < fl.size(); i++) {
        const bool first = i == 0;
        if ((s = launch_fft(fl[i], false, first, first ? (const void*)Sa : Wa, first ? (1ull << P.ma) : T.H, Wa, PL, ds, st)) != GF2X_OK)
            return s;
        if ((s = launch_fft(fl[i], false, first, first ? (const void*)Sb : Wb, first ? (1ull << P.mb) : T.H, Wb, PL, ds, st)) != GF2X_OK)
            return s;
    }
    if (fl.size() == 1) return fail(GF2X_EINVAL, "truncated path needs a table pass");   // (m - 1 >= 13 always has one)
    {
        BottomParams bp;
        bp.A = Wa; bp.B = Wb;
        bp.total = T.H;
        bp.ntiles = (T.H + (1ull << BT_BITS) - 1) >> BT_BITS;
        bp.m = T.m - 1; bp.L = fl.back().layers; bp.mode = 7; bp.map = IdxMap{0, 0, 0};
        ProfScope ps("k_bottom", 48.0 * T.H, st, (double)bp.ntiles * (3.0 * bp.L * 128.0 + 576.0) * OPS_BS_MUL32);
        bottom_launch(bp, smc, st);
    }
    for (size_t i = fl.size() - 1; i-- > 0;)
        if ((s = launch_fft(fl[i], true, false, Wa, T.H, Wa, PL, ds, st)) != GF2X_OK) return s;
    // g_hi = iFFT_j(...) + Reduce(g_lo)[0, 2^j): Reduce on a copy of g_lo (Wb's lower half is free now)
    CUDA_TRY(cudaMemcpyAsync(Wb, Wa, T.H * 16, cudaMemcpyDeviceToDevice, st));
    if ((s = reduce(Wb, nullptr)) != GF2X_OK) return s;
    {
        ProfScope ps("k_xor_range", 48.0 * T.U, st);
        k_xor_range<<<grid_for(T.U, 256, smc, 8), 256, 0, st>>>(Ua - 0, Wb - 0, 0, T.U);
    }
    const uint64_t n_out = P.na + P.nb;
    if ((s = check_launch("trunc combine")) != GF2X_OK) return s;
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
        k_ipsi_bs<<<grid_for((n_out + IB_TILE - 1) / IB_TILE, 1, smc, 2), IB_THREADS, 6 * IB_TILE * 4, st>>>(Wa, ds->tabs, P.N,
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
