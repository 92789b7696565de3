// frob.cuh -- App. C building block: BasisCvt / iBasisCvt on GF(2)
// coefficients ("The basis conversion can be proceeded straightforwardly with alg. 3"), the first
// step of the multiply through the Frobenius bijection.  Included by gf2x.cu.
//
// The coefficients are packed 64 per word (bit t of the polynomial = bit t % 64 of word t / 64).  Alg. 3's
// Taylor steps (Alg. 2, the same (lg, K) list as the word-level conversion, in the inner-first order of
// DESIGN.md R14) act on bit positions: step (lg, K) on every segment of 2^lg bits, h = 2^(lg-1), u = h >> K,
// d = h - u, "f[i - d] ^= f[i] for i = 2h-1 .. h" splits into two parallel sweeps (the targets of one sweep
// are never its sources):
//   sweep 1: targets [h, h + u)  (sources [2h - u, 2h));   sweep 2: targets [u, h)  (sources [h, 2h - u)),
// forward in the order 1, 2 and inverse (ascending i) in the order 2, 1.  One thread owns one word: it
// XORs in the source bits (a funnel shift of the words d bits up) under the mask of its target bits; words
// that hold no targets are not touched.  This is the plain form of the step (one HBM sweep each); the tiled
// forms of the word-level conversion are the next step for it.
#pragma once

__global__ void __launch_bounds__(256) k_bitcvt_sweep(uint64_t* __restrict__ G, uint64_t nw, int lg, uint64_t d,
                                                      uint64_t tlo, uint64_t thi, uint64_t pmask) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
        if (lg < 6) {   // segments inside the word: a periodic mask, sources in the same word
            const uint64_t x = G[w];
            G[w] = x ^ ((x >> d) & pmask);
            continue;
        }
        const uint64_t len = 1ull << lg, o = (w << 6) & (len - 1);   // the word's offset in its segment
        const uint64_t lo = tlo > o ? tlo - o : 0, hi = thi < o + 64 ? thi - o : 64;
        if (thi <= o || tlo >= o + 64 || lo >= hi) continue;
        const uint64_t mask = (hi >= 64 ? ~0ull : ((1ull << hi) - 1)) & ~((1ull << lo) - 1);
        const uint64_t sp = (w << 6) + d, w0 = sp >> 6;
        const int sh = (int)(sp & 63);
        uint64_t src = G[w0] >> sh;
        if (sh && w0 + 1 < nw) src |= G[w0 + 1] << (64 - sh);
        G[w] ^= src & mask;
    }
}

static gf2x_status run_bitcvt(uint64_t* G, int M, bool inverse, int smc, cudaStream_t st) {
    std::vector<CvtOp> ops;
    cvt_ops(M, 0, ops);
    if (inverse) std::reverse(ops.begin(), ops.end());
    const uint64_t nw = 1ull << (M - 6);
    for (const CvtOp& op : ops) {
        const uint64_t h = 1ull << (op.lg - 1), u = h >> op.K, d = h - u;
        for (int sw = 0; sw < 2; sw++) {
            const bool first = inverse ? sw == 1 : sw == 0;   // sweep 1 (targets [h, h+u)) or sweep 2 ([u, h))
            const uint64_t tlo = first ? h : u, thi = first ? h + u : h;
            uint64_t pmask = 0;
            if (op.lg < 6)
                for (uint64_t seg = 0; seg < 64; seg += 2 * h)
                    for (uint64_t t = tlo; t < thi; t++) pmask |= 1ull << (seg + t);
            ProfScope ps("k_bitcvt_sweep", 16.0 * nw, st);
            k_bitcvt_sweep<<<grid_for(nw, 256, smc, 8), 256, 0, st>>>(G, nw, op.lg, d, tlo, thi, pmask);
        }
    }
    return check_launch("bit-level BasisCvt");
}
