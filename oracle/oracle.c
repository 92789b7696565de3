/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for arXiv 1708.09746
 * ("Faster Multiplication for Long Binary Polynomials", Chen, Cheng, Kuo, Li, Yang).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA product path (paper_1708_09746_b200/), and neither side imports the other.
 *
 * Citations: "P:a-b" = lines of PAPER.md (the paper's LaTeX source), with section / algorithm.
 *
 * Contents (SURVEY.md §8c numbering):
 *   O2  carry-less word multiply: shift-and-xor clmul64 (or the x86 PCLMULQDQ instruction when the
 *       CPU has it -- or_clmul_impl() says which), schoolbook, Karatsuba, single-output-word.
 *       Definition: c_k = XOR_{i+j=k} a_i b_j.
 *   O3  the paper's Alg. 5 step by step:
 *         tower field TGF(2^128) (Def. of v_k P:658-665), Karatsuba per level
 *         (sec 4.1.3), bottoming out at GF(256) log/exp tables that are
 *         themselves derived from the bit-level recursion;
 *         subspace vanishing polynomials s_k via s_{k+1} = s_k^2 + s_k (corollary P:718-721);
 *         GF(2^128) = GF(2)[z]/(z^128+z^7+z^2+z+1) (sec 2.2.1) and the isomorphism
 *         changeRepr (sec 4.3) fixed by the deterministic rule of DESIGN.md R9;
 *         BasisCvt = Alg. 3 with VarSubs = Alg. 2, iBasisCvt (R7);
 *         FFT_LCH = Alg. 1, iFFT (R8); pointmul; InterleavedCombine.
 *       w = 128 variant (sec 4.2): TGF(2^256) one tower level up, GF(2^256) modulo
 *       z^256+z^10+z^5+z^2+1 (R20) and changeRepr_256 by the same rule, Alg. 5 on 128-bit blocks.
 *       Alg. 4 (sec 3.1): FFT_LCH in GF(2^128) polynomial basis, dense multipliers psi^-1(s_k).
 *       App. C: multiplication through the Frobenius bijection E_(beta_(m+64) + V_m):
 *       BasisCvt on GF(2) coefficients, the 7-layer encoding, FFT_LCH displaced by beta_(m+64), decoding.
 *   O4  product check modulo random irreducible degree-64 polynomials.
 *
 * All arithmetic is exact (GF(2) AND/XOR); no floating point anywhere.
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>
#if defined(__x86_64__)
#include <immintrin.h>
#include <cpuid.h>
#endif
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------------------------ */
/* O2: carry-less multiplication (the definition c_k = XOR_{i+j=k} a_i b_j)         */
/* ------------------------------------------------------------------------------------------ */

/* Shift-and-xor: for every set bit i of a, add b * x^i. */
static u128 clmul64_portable(uint64_t a, uint64_t b) {
    u128 acc = 0;
    for (int i = 0; i < 64; i++)
        if ((a >> i) & 1) acc ^= ((u128)b) << i;
    return acc;
}

#if defined(__x86_64__)
__attribute__((target("pclmul,sse4.1")))
static u128 clmul64_hw(uint64_t a, uint64_t b) {
    __m128i x = _mm_set_epi64x(0, (long long)a);
    __m128i y = _mm_set_epi64x(0, (long long)b);
    __m128i z = _mm_clmulepi64_si128(x, y, 0x00);
    uint64_t lo = (uint64_t)_mm_cvtsi128_si64(z);
    uint64_t hi = (uint64_t)_mm_extract_epi64(z, 1);
    return ((u128)hi << 64) | lo;
}
static int have_pclmul(void) {
    unsigned a, b, c, d;
    if (!__get_cpuid(1, &a, &b, &c, &d)) return 0;
    return (c & bit_PCLMUL) != 0;
}
#endif

static int g_use_hw = -1; /* -1 unknown, 0 portable, 1 PCLMULQDQ */

static void clmul_init(void) {
    if (g_use_hw >= 0) return;
#if defined(__x86_64__)
    g_use_hw = have_pclmul();
#else
    g_use_hw = 0;
#endif
}

static inline u128 clmul64(uint64_t a, uint64_t b) {
#if defined(__x86_64__)
    if (g_use_hw == 1) return clmul64_hw(a, b);
#endif
    return clmul64_portable(a, b);
}

/* 1 if PCLMULQDQ is used behind clmul64, 0 if the shift-and-xor loop is. Forcing: mode 0/1. */
int or_clmul_impl(void) { clmul_init(); return g_use_hw; }
void or_clmul_force_portable(int portable) { clmul_init(); if (portable) g_use_hw = 0; }

void or_clmul64(uint64_t a, uint64_t b, uint64_t *lo, uint64_t *hi) {
    clmul_init();
    u128 r = clmul64(a, b);
    *lo = (uint64_t)r; *hi = (uint64_t)(r >> 64);
}
void or_clmul64_portable(uint64_t a, uint64_t b, uint64_t *lo, uint64_t *hi) {
    u128 r = clmul64_portable(a, b);
    *lo = (uint64_t)r; *hi = (uint64_t)(r >> 64);
}

/* Schoolbook: c (na+nb words) = XOR over all word pairs (i,j) of clmul(a_i,b_j) * x^(64(i+j)). */
void or_mul_schoolbook(const uint64_t *a, size_t na, const uint64_t *b, size_t nb, uint64_t *c) {
    clmul_init();
    memset(c, 0, (na + nb) * sizeof(uint64_t));
    for (size_t i = 0; i < na; i++) {
        if (!a[i]) continue;
        for (size_t j = 0; j < nb; j++) {
            u128 p = clmul64(a[i], b[j]);
            c[i + j] ^= (uint64_t)p;
            c[i + j + 1] ^= (uint64_t)(p >> 64);
        }
    }
}

/* Karatsuba on n words (any n): a = a0 + x^(64h) a1, b likewise, h = ceil(n/2):
 * a*b = a0b0 + x^(64h) [(a0+a1)(b0+b1) + a0b0 + a1b1] + x^(128h) a1b1.
 * c must hold 2n words. Below 32 words it falls back to schoolbook. */
static void kara_rec(const uint64_t *a, const uint64_t *b, size_t n, uint64_t *c, uint64_t *tmp) {
    if (n <= 32) { or_mul_schoolbook(a, n, b, n, c); return; }
    size_t h = (n + 1) / 2, l = n - h;          /* low part h words, high part l words (l <= h) */
    uint64_t *sa = tmp, *sb = tmp + h, *mid = tmp + 2 * h, *rest = tmp + 4 * h;
    kara_rec(a, b, h, c, rest);                  /* c[0, 2h)      = a0 b0 */
    memset(c + 2 * h, 0, (2 * n - 2 * h) * sizeof(uint64_t));
    if (l == h) {
        kara_rec(a + h, b + h, l, c + 2 * h, rest); /* c[2h, 2n) = a1 b1 */
    } else {
        /* l < h: multiply the unequal high parts by schoolbook (only happens for odd n) */
        or_mul_schoolbook(a + h, l, b + h, l, c + 2 * h);
    }
    for (size_t i = 0; i < h; i++) {
        sa[i] = a[i] ^ (i < l ? a[h + i] : 0);
        sb[i] = b[i] ^ (i < l ? b[h + i] : 0);
    }
    kara_rec(sa, sb, h, mid, rest);              /* mid = (a0+a1)(b0+b1), 2h words */
    for (size_t i = 0; i < 2 * h; i++) mid[i] ^= c[i];                     /* - a0b0 */
    for (size_t i = 0; i < 2 * l; i++) mid[i] ^= c[2 * h + i];             /* - a1b1 */
    for (size_t i = 0; i < 2 * h; i++) c[h + i] ^= mid[i];
}

/* c (2n words) = a * b, both n words. */
void or_mul_karatsuba(const uint64_t *a, const uint64_t *b, size_t n, uint64_t *c) {
    clmul_init();
    if (n == 0) return;
    /* scratch: at each level 4h + rest; bounded by 8n + small */
    uint64_t *tmp = (uint64_t *)calloc(8 * n + 256, sizeof(uint64_t));
    kara_rec(a, b, n, c, tmp);
    free(tmp);
}

/* Single output word w of a*b: c_w = XOR_{i+j=w} lo(a_i b_j) ^ XOR_{i+j=w-1} hi(a_i b_j). O(n). */
uint64_t or_mul_word(const uint64_t *a, size_t na, const uint64_t *b, size_t nb, size_t w) {
    clmul_init();
    uint64_t r = 0;
    for (size_t i = 0; i < na && i <= w; i++) {
        size_t j = w - i;
        if (j < nb) r ^= (uint64_t)clmul64(a[i], b[j]);
        if (j >= 1 && j - 1 < nb) r ^= (uint64_t)(clmul64(a[i], b[j - 1]) >> 64);
    }
    return r;
}

/* ------------------------------------------------------------------------------------------ */
/* O3 part 1: the tower field TGF(2^(2^l)) in the basis (v_k)                    */
/*   TGF(2^2) = GF(2)[x1]/(x1^2+x1+1);  TGF(2^(2^l)) = TGF(2^(2^(l-1)))[x_l]/(x_l^2+x_l+P)      */
/*   with P = x_1 ... x_(l-1) = v_(2^(l-1)-1).  An element is the integer whose bit k is the     */
/*   coordinate of v_k = prod x_(j+1)^(b_j) (Def. v_k).  Its upper half is the        */
/*   coefficient of x_l since v_(2^(l-1)+j) = x_l v_j.                                           */
/* ------------------------------------------------------------------------------------------ */

/* Pure recursion down to GF(2) = AND.  (a0 + a1 X)(b0 + b1 X), X^2 = X + P:
 *   lo = a0b0 + a1b1 P,  hi = (a0+a1)(b0+b1) + a0b0   (Karatsuba, sec 4.1.3). */
static u128 tmul_bits(u128 a, u128 b, int l) {
    if (l == 0) return a & b & 1;
    int h = 1 << (l - 1);
    u128 mask = (((u128)1) << h) - 1;
    u128 a0 = a & mask, a1 = a >> h, b0 = b & mask, b1 = b >> h;
    u128 P = ((u128)1) << (h - 1);           /* v_(2^(l-1)-1); = 1 for l = 1 */
    u128 p0 = tmul_bits(a0, b0, l - 1);
    u128 p2 = tmul_bits(a1, b1, l - 1);
    u128 p1 = tmul_bits(a0 ^ a1, b0 ^ b1, l - 1);
    u128 lo = p0 ^ tmul_bits(p2, P, l - 1);
    u128 hi = p1 ^ p0;
    return lo | (hi << h);
}

/* GF(256) = TGF(2^8) log/exp tables (P:1073-1075 uses log/exp tables for the smallest fields),
 * built from tmul_bits with the smallest generator of order 255 (SPEC S:207 rule). */
static uint8_t g_exp[512];
static int g_log[256];
static int g_tables_ready = 0;
static int g_generator = 0;

static void tower_init(void) {
    if (g_tables_ready) return;
    for (int g = 2; g < 256; g++) {
        int x = 1, ord = 0;
        do { x = (int)tmul_bits((u128)x, (u128)g, 3); ord++; } while (x != 1 && ord < 300);
        if (ord == 255) { g_generator = g; break; }
    }
    int x = 1;
    for (int i = 0; i < 255; i++) {
        g_exp[i] = (uint8_t)x; g_exp[i + 255] = (uint8_t)x;
        g_log[x] = i;
        x = (int)tmul_bits((u128)x, (u128)g_generator, 3);
    }
    g_exp[510] = g_exp[0]; g_exp[511] = g_exp[1];
    g_log[0] = -1;
    g_tables_ready = 1;
}

/* Tower product at level l (2^l-bit elements, l <= 7), recursion bottoming out at GF(256).
 * Elements of a subfield are the small integers, so levels 0..3 all use the GF(256)
 * table.  If one operand lies in the half-size subfield (b1 == 0 or a1 == 0) the recursion drops
 * to 2 half-size products: Prop. 2 falling out of the formula. */
static u128 tmul(u128 a, u128 b, int l) {
    if (l <= 3) {
        unsigned x = (unsigned)a, y = (unsigned)b;
        if (!x || !y) return 0;
        return g_exp[g_log[x] + g_log[y]];
    }
    int h = 1 << (l - 1);
    u128 mask = (((u128)1) << h) - 1;
    u128 a0 = a & mask, a1 = a >> h, b0 = b & mask, b1 = b >> h;
    if (b1 == 0) return tmul(a0, b0, l - 1) | (tmul(a1, b0, l - 1) << h);
    if (a1 == 0) return tmul(a0, b0, l - 1) | (tmul(a0, b1, l - 1) << h);
    u128 P = ((u128)1) << (h - 1);
    u128 p0 = tmul(a0, b0, l - 1);
    u128 p2 = tmul(a1, b1, l - 1);
    u128 p1 = tmul(a0 ^ a1, b0 ^ b1, l - 1);
    u128 lo = p0 ^ tmul(p2, P, l - 1);
    u128 hi = p1 ^ p0;
    return lo | (hi << h);
}

static inline u128 mk(uint64_t lo, uint64_t hi) { return ((u128)hi << 64) | lo; }
static inline void unmk(u128 x, uint64_t *out) { out[0] = (uint64_t)x; out[1] = (uint64_t)(x >> 64); }

/* Exported tower multiply: a, b, r are 2-word little-endian 128-bit values. */
void or_tower_mul(const uint64_t *a, const uint64_t *b, int level, uint64_t *r) {
    tower_init();
    unmk(tmul(mk(a[0], a[1]), mk(b[0], b[1]), level), r);
}
void or_tower_mul_bits(const uint64_t *a, const uint64_t *b, int level, uint64_t *r) {
    unmk(tmul_bits(mk(a[0], a[1]), mk(b[0], b[1]), level), r);
}
int or_gf256_generator(void) { tower_init(); return g_generator; }

/* ------------------------------------------------------------------------------------------ */
/* O3 part 2: subspace vanishing polynomials s_k (Def. 2)                           */
/*   s_0(x) = x, s_(k+1)(x) = s_k(x)^2 + s_k(x)  (recursivity corollary P:718-721),            */
/*   i.e. s_k = s_1 applied k times with s_1(x) = x (x) x + x.                                  */
/* ------------------------------------------------------------------------------------------ */
static inline u128 s1(u128 x) { return tmul(x, x, 7) ^ x; }

static u128 s_eval(int k, u128 x) {
    for (int i = 0; i < k; i++) x = s1(x);
    return x;
}
void or_s_eval(int k, const uint64_t *x, uint64_t *r) { tower_init(); unmk(s_eval(k, mk(x[0], x[1])), r); }

/* ------------------------------------------------------------------------------------------ */
/* O3 part 3: GF(2^128) in polynomial basis (sec 2.2.1) and changeRepr             */
/* ------------------------------------------------------------------------------------------ */
/* multiply by z modulo z^128 + z^7 + z^2 + z + 1 */
static inline u128 gf128_mulz(u128 a) {
    int carry = (int)(a >> 127);
    a <<= 1;
    if (carry) a ^= 0x87;
    return a;
}
/* Shift-and-add: for every set bit i of b, add a * z^i mod g. */
static u128 gf128_mul(u128 a, u128 b) {
    u128 acc = 0;
    for (int i = 0; i < 128; i++) {
        if ((b >> i) & 1) acc ^= a;
        a = gf128_mulz(a);
    }
    return acc;
}
void or_gf128_mul(const uint64_t *a, const uint64_t *b, uint64_t *r) {
    unmk(gf128_mul(mk(a[0], a[1]), mk(b[0], b[1])), r);
}

/* Solve r^2 + r = c in GF(2^128) by Gaussian elimination on the GF(2)-linear map L(x) = x^2 + x
 * (its kernel is {0, 1}).  Returns 0 and the numerically smaller root, or -1 if no root. */
static int gf128_solve_as(u128 c, u128 *root) {
    u128 col[128];
    for (int i = 0; i < 128; i++) { u128 e = ((u128)1) << i; col[i] = gf128_mul(e, e) ^ e; }
    /* augmented system: rows = output bits; we do elimination on columns stored as bit-vectors
     * by transposing into row form: row r = (bits of column images at position r | rhs bit r) */
    u128 row[128]; int rhs[128];
    for (int r = 0; r < 128; r++) {
        u128 v = 0;
        for (int i = 0; i < 128; i++) if ((col[i] >> r) & 1) v |= ((u128)1) << i;
        row[r] = v; rhs[r] = (int)((c >> r) & 1);
    }
    int pivcol[128]; int nr = 0;
    for (int cidx = 0; cidx < 128 && nr < 128; cidx++) {
        int p = -1;
        for (int r = nr; r < 128; r++) if ((row[r] >> cidx) & 1) { p = r; break; }
        if (p < 0) continue;
        u128 t = row[p]; row[p] = row[nr]; row[nr] = t;
        int tr = rhs[p]; rhs[p] = rhs[nr]; rhs[nr] = tr;
        for (int r = 0; r < 128; r++)
            if (r != nr && ((row[r] >> cidx) & 1)) { row[r] ^= row[nr]; rhs[r] ^= rhs[nr]; }
        pivcol[nr] = cidx; nr++;
    }
    for (int r = nr; r < 128; r++) if (rhs[r]) return -1;   /* inconsistent */
    u128 x = 0;  /* free variables = 0 */
    for (int r = 0; r < nr; r++) if (rhs[r]) x |= ((u128)1) << pivcol[r];
    u128 alt = x ^ 1;  /* the other root (kernel {0,1}) */
    *root = (alt < x) ? alt : x;
    return 0;
}

/* changeRepr (sec 4.3): Mcol[k] = image in GF(2^128) of tower basis element v_k, k < 128.
 * Rule (R9): X_1^2+X_1 = 1, X_k^2+X_k = X_1...X_(k-1) (the defining relations P:643-650),
 * each the numerically smaller root; v_k -> prod_{bit j of k} X_(j+1).
 * psi_inv = Mcol (tower -> polynomial basis); psi = Mcol^(-1). */
static u128 g_Mcol[128], g_psicol[128];
static u128 g_X[8];
static int g_psi_ready = 0;

static int psi_init(void) {
    if (g_psi_ready) return 0;
    u128 prod = 1;
    for (int k = 1; k <= 7; k++) {
        if (gf128_solve_as(prod, &g_X[k]) != 0) return -1;
        prod = gf128_mul(prod, g_X[k]);
    }
    for (int k = 0; k < 128; k++) {
        u128 v = 1;
        for (int j = 0; j < 7; j++) if ((k >> j) & 1) v = gf128_mul(v, g_X[j + 1]);
        g_Mcol[k] = v;
    }
    /* invert M: Gauss-Jordan on [M | I] with M given by columns -> work on rows */
    u128 A[128], B[128];
    for (int r = 0; r < 128; r++) {
        u128 v = 0;
        for (int c = 0; c < 128; c++) if ((g_Mcol[c] >> r) & 1) v |= ((u128)1) << c;
        A[r] = v; B[r] = ((u128)1) << r;
    }
    for (int c = 0; c < 128; c++) {
        int p = -1;
        for (int r = c; r < 128; r++) if ((A[r] >> c) & 1) { p = r; break; }
        if (p < 0) return -2;
        u128 t = A[p]; A[p] = A[c]; A[c] = t; t = B[p]; B[p] = B[c]; B[c] = t;
        for (int r = 0; r < 128; r++)
            if (r != c && ((A[r] >> c) & 1)) { A[r] ^= A[c]; B[r] ^= B[c]; }
    }
    /* now A = I, rows of B = rows of M^-1; psi column c = M^-1 e_c */
    for (int c = 0; c < 128; c++) {
        u128 v = 0;
        for (int r = 0; r < 128; r++) if ((B[r] >> c) & 1) v |= ((u128)1) << r;
        g_psicol[c] = v;
    }
    g_psi_ready = 1;
    return 0;
}

static u128 apply_cols(const u128 *cols, u128 x) {
    u128 r = 0;
    for (int i = 0; i < 128; i++) if ((x >> i) & 1) r ^= cols[i];
    return r;
}
static inline u128 psi(u128 x) { return apply_cols(g_psicol, x); }      /* poly -> tower */
static inline u128 psi_inv(u128 x) { return apply_cols(g_Mcol, x); }   /* tower -> poly */

int or_psi_init(void) { return psi_init(); }
void or_psi(const uint64_t *x, uint64_t *r) { psi_init(); unmk(psi(mk(x[0], x[1])), r); }
void or_psi_inv(const uint64_t *x, uint64_t *r) { psi_init(); unmk(psi_inv(mk(x[0], x[1])), r); }
void or_psi_generator(int k, uint64_t *r) { psi_init(); unmk(g_X[k], r); }
/* columns of psi (128 x 2 words) -- images of z^0..z^127 in the tower */
void or_psi_columns(uint64_t *out) { psi_init(); for (int i = 0; i < 128; i++) unmk(g_psicol[i], out + 2 * i); }

/* ------------------------------------------------------------------------------------------ */
/* O3 part 4: BasisCvt (Alg. 3) via VarSubs (Alg. 2), and its inverse    */
/* Arrays of 128-bit units (a 64-bit block occupies the low half).  XOR only.       */
/* ------------------------------------------------------------------------------------------ */

/* Alg. 2 division by y^k' = x^(2^(l-1)) + x^(2^(l-1-K)) of one segment of len = 2^(l+sigma) words,
 * "by repeatedly subtracting": for i = len-1 down to h, f[i-d] ^= f[i], d = h - h>>K. */
/* optional trace of the Taylor steps (for the App. B pin): (len, K, d, xor count) per call */
static long *g_trace = NULL; static int g_trace_n = 0, g_trace_max = 0;
static void trace_step(size_t len, int K, size_t d, size_t xors) {
    if (!g_trace || g_trace_n >= g_trace_max) return;
    long *t = g_trace + 4 * g_trace_n++;
    t[0] = (long)len; t[1] = K; t[2] = (long)d; t[3] = (long)xors;
}
static void taylor(u128 *f, size_t s, size_t len, int K) {
    size_t h = len / 2, d = h - (h >> K);
    trace_step(len, K, d, h);
    for (size_t i = len - 1; i >= h; i--) {
        f[s + i - d] ^= f[s + i];
        if (i == h) break;
    }
}
static void itaylor(u128 *f, size_t s, size_t len, int K) {
    size_t h = len / 2, d = h - (h >> K);
    for (size_t i = h; i < len; i++) f[s + i - d] ^= f[s + i];
}

static int floor_log2(int x) { int r = 0; while ((1 << (r + 1)) <= x) r++; return r; }

/* CVT(f, base, m, sigma): convert the 2^m units of 2^sigma words starting at base (R4-R6). */
static void cvt(u128 *f, size_t base, int m, int sigma) {
    if (m <= 1) return;                                   /* deg <= 1: g = f (Alg. 3 line 1) */
    int K = 1 << floor_log2(m - 1);                       /* largest power of two with 2^K <= deg */
    for (int l = m; l >= K + 1; l--)                      /* VarSubs(f, y = s_K(x)) */
        for (size_t s = 0; s < ((size_t)1 << (m + sigma)); s += ((size_t)1 << (l + sigma)))
            taylor(f, base + s, (size_t)1 << (l + sigma), K);
    cvt(f, base, m - K, sigma + K);                       /* BasisCvt(h(y)) over y (outer) */
    for (size_t c = 0; c < ((size_t)1 << (m + sigma)); c += ((size_t)1 << (K + sigma)))
        cvt(f, base + c, K, sigma);                       /* BasisCvt(q_i(x)) (inner) */
}
static void icvt(u128 *f, size_t base, int m, int sigma) {
    if (m <= 1) return;
    int K = 1 << floor_log2(m - 1);
    for (size_t c = 0; c < ((size_t)1 << (m + sigma)); c += ((size_t)1 << (K + sigma)))
        icvt(f, base + c, K, sigma);
    icvt(f, base, m - K, sigma + K);
    for (int l = K + 1; l <= m; l++)
        for (size_t s = 0; s < ((size_t)1 << (m + sigma)); s += ((size_t)1 << (l + sigma)))
            itaylor(f, base + s, (size_t)1 << (l + sigma), K);
}

/* Exported on arrays of n = 2^m units of `w` 64-bit words each (w = 1 or 2). */
static void to128(const uint64_t *in, size_t n, int w, u128 *f) {
    for (size_t i = 0; i < n; i++) f[i] = (w == 1) ? (u128)in[i] : mk(in[2 * i], in[2 * i + 1]);
}
static void from128(const u128 *f, size_t n, int w, uint64_t *out) {
    for (size_t i = 0; i < n; i++) { if (w == 1) out[i] = (uint64_t)f[i]; else unmk(f[i], out + 2 * i); }
}
void or_basis_cvt(uint64_t *data, int m, int w) {
    size_t n = (size_t)1 << m;
    u128 *f = (u128 *)malloc(n * sizeof(u128));
    to128(data, n, w, f); cvt(f, 0, m, 0); from128(f, n, w, data);
    free(f);
}
/* record the Taylor steps BasisCvt performs on 2^m units: 4 longs per step; returns the count */
int or_cvt_trace(int m, long *out, int max_steps) {
    size_t n = (size_t)1 << m;
    u128 *f = (u128 *)calloc(n, sizeof(u128));
    g_trace = out; g_trace_n = 0; g_trace_max = max_steps;
    cvt(f, 0, m, 0);
    int cnt = g_trace_n;
    g_trace = NULL;
    free(f);
    return cnt;
}
void or_ibasis_cvt(uint64_t *data, int m, int w) {
    size_t n = (size_t)1 << m;
    u128 *f = (u128 *)malloc(n * sizeof(u128));
    to128(data, n, w, f); icvt(f, 0, m, 0); from128(f, n, w, data);
    free(f);
}

/* ------------------------------------------------------------------------------------------ */
/* O3 part 5: FFT_LCH (Alg. 1) at alpha = 0 over the tower, and its inverse   */
/*   layer k = m-1 .. 0, block base b (multiple of 2^(k+1)), c = s_k(phi_v(b)):                 */
/*     A[b+i] ^= c (x) A[b+2^k+i];  A[b+2^k+i] ^= A[b+i]      (second multiplier s_k(v_k) = 1,   */
/*   Prop. 1).  Output i = f(phi_v(i)) (R2).                                 */
/*   c is computed as s_k(phi_v(b)) = s_1(s_(k-1)(phi_v(b))), cached per block (SURVEY c.2 O3).  */
/* ------------------------------------------------------------------------------------------ */

/* mult[b >> (k+1)] for layer k, built bottom-up: layer 0 constants are phi_v(b) = b itself. */
static void layer_constants(int m, int k, u128 *prev, u128 *out) {
    size_t nb = (size_t)1 << (m - k - 1);
    if (k == 0) { for (size_t j = 0; j < nb; j++) out[j] = (u128)(j << 1); return; }
    /* block j of layer k has base b = j * 2^(k+1), which is block 2j of layer k-1 */
    for (size_t j = 0; j < nb; j++) out[j] = s1(prev[2 * j]);
}

static u128 **all_constants(int m) {
    u128 **C = (u128 **)calloc((size_t)(m > 0 ? m : 1), sizeof(u128 *));
    for (int k = 0; k < m; k++) {
        C[k] = (u128 *)malloc(((size_t)1 << (m - k - 1)) * sizeof(u128));
        layer_constants(m, k, k ? C[k - 1] : NULL, C[k]);
    }
    return C;
}
static void free_constants(u128 **C, int m) { for (int k = 0; k < m; k++) free(C[k]); free(C); }

static void fft(u128 *A, int m, u128 **C) {
    for (int k = m - 1; k >= 0; k--) {
        size_t half = (size_t)1 << k, nb = (size_t)1 << (m - k - 1);
#pragma omp parallel for schedule(static) if (nb * half >= 4096)
        for (size_t j = 0; j < nb; j++) {
            size_t b = j << (k + 1);
            u128 c = C[k][j];
            for (size_t i = 0; i < half; i++) {
                A[b + i] ^= tmul(A[b + half + i], c, 7);
                A[b + half + i] ^= A[b + i];
            }
        }
    }
}
static void ifft(u128 *A, int m, u128 **C) {
    for (int k = 0; k < m; k++) {
        size_t half = (size_t)1 << k, nb = (size_t)1 << (m - k - 1);
#pragma omp parallel for schedule(static) if (nb * half >= 4096)
        for (size_t j = 0; j < nb; j++) {
            size_t b = j << (k + 1);
            u128 c = C[k][j];
            for (size_t i = 0; i < half; i++) {
                A[b + half + i] ^= A[b + i];
                A[b + i] ^= tmul(A[b + half + i], c, 7);
            }
        }
    }
}

void or_fft(uint64_t *data, int m) {
    tower_init();
    size_t n = (size_t)1 << m;
    u128 *A = (u128 *)malloc(n * sizeof(u128));
    u128 **C = all_constants(m);
    to128(data, n, 2, A); fft(A, m, C); from128(A, n, 2, data);
    free_constants(C, m); free(A);
}
void or_ifft(uint64_t *data, int m) {
    tower_init();
    size_t n = (size_t)1 << m;
    u128 *A = (u128 *)malloc(n * sizeof(u128));
    u128 **C = all_constants(m);
    to128(data, n, 2, A); ifft(A, m, C); from128(A, n, 2, data);
    free_constants(C, m); free(A);
}
/* layer constant s_k(phi_v(b)) for block index j (b = j << (k+1)) of an m-layer FFT */
void or_fft_constant(int m, int k, uint64_t j, uint64_t *r) {
    tower_init();
    u128 **C = all_constants(m);
    unmk(C[k][j], r);
    free_constants(C, m);
}
/* number of non-trivial multiplications (constant != 0 and != 1) issued by fft() on m layers
 * with the top layer acting on nonzero upper halves: used to check the 1/2 n log n bound */
uint64_t or_fft_mult_count(int m) {
    tower_init();
    u128 **C = all_constants(m);
    uint64_t cnt = 0;
    for (int k = 0; k < m; k++)
        for (size_t j = 0; j < ((size_t)1 << (m - k - 1)); j++)
            if (C[k][j] > 1) cnt += (uint64_t)1 << k;
    free_constants(C, m);
    return cnt;
}

/* ------------------------------------------------------------------------------------------ */
/* O3 part 6: Alg. 5 binPolyMul, w = 64                                           */
/* ------------------------------------------------------------------------------------------ */
static int ceil_log2_sz(size_t x) { int r = 0; while (((size_t)1 << r) < x) r++; return r; }

/* Stage dump buffers (optional, may be NULL): each N x 2 words.
 *   st_cvt_a/b : after BasisCvt + changeRepr (tower, novel basis)   -- Alg. 5 lines 3-6
 *   st_fft_a/b : after FFT_LCH                                       -- lines 7-8
 *   st_prod    : after pointmul                                      -- line 9
 *   st_ifft    : after iFFT                                          -- line 10
 *   st_icvt    : after iBasisCvt (tower)                             -- line 11
 * c receives na+nb words (R13).  Returns 0, or a negative code on an internal
 * assertion failure (bit 127 set, nonzero coefficient above L). */
int or_alg5_mul(const uint64_t *a, uint64_t a_bits, const uint64_t *b, uint64_t b_bits, uint64_t *c,
                uint64_t *st_cvt_a, uint64_t *st_cvt_b, uint64_t *st_fft_a, uint64_t *st_fft_b,
                uint64_t *st_prod, uint64_t *st_ifft, uint64_t *st_icvt) {
    tower_init();
    if (psi_init() != 0) return -10;
    size_t na = (a_bits + 63) / 64, nb = (b_bits + 63) / 64;
    if (a_bits == 0 || b_bits == 0) { memset(c, 0, (na + nb) * sizeof(uint64_t)); return 0; }
    size_t L = na + nb - 1;
    int m = ceil_log2_sz(L);
    size_t N = (size_t)1 << m;
    u128 *A = (u128 *)calloc(N, sizeof(u128));
    u128 *B = (u128 *)calloc(N, sizeof(u128));
    /* Split: with w = 64 and little-endian words this is a copy; mask bits >= a_bits */
    for (size_t j = 0; j < na; j++) {
        uint64_t w = a[j];
        if (j == na - 1 && (a_bits & 63)) w &= (((uint64_t)1) << (a_bits & 63)) - 1;
        A[j] = w;
    }
    for (size_t j = 0; j < nb; j++) {
        uint64_t w = b[j];
        if (j == nb - 1 && (b_bits & 63)) w &= (((uint64_t)1) << (b_bits & 63)) - 1;
        B[j] = w;
    }
    /* BasisCvt on the 64-bit blocks, before changeRepr */
    cvt(A, 0, m, 0); cvt(B, 0, m, 0);
    /* changeRepr */
#pragma omp parallel for schedule(static) if (N >= 4096)
    for (size_t i = 0; i < N; i++) { A[i] = psi(A[i]); B[i] = psi(B[i]); }
    if (st_cvt_a) from128(A, N, 2, st_cvt_a);
    if (st_cvt_b) from128(B, N, 2, st_cvt_b);
    /* FFT_LCH at alpha = 0 */
    u128 **C = all_constants(m);
    fft(A, m, C); fft(B, m, C);
    if (st_fft_a) from128(A, N, 2, st_fft_a);
    if (st_fft_b) from128(B, N, 2, st_fft_b);
    /* pointmul */
#pragma omp parallel for schedule(static) if (N >= 4096)
    for (size_t i = 0; i < N; i++) A[i] = tmul(A[i], B[i], 7);
    if (st_prod) from128(A, N, 2, st_prod);
    /* iFFT_LCH */
    ifft(A, m, C);
    if (st_ifft) from128(A, N, 2, st_ifft);
    /* iBasisCvt in the tower representation */
    icvt(A, 0, m, 0);
    if (st_icvt) from128(A, N, 2, st_icvt);
    /* changeRepr back */
    int err = 0;
#pragma omp parallel for schedule(static) if (N >= 4096)
    for (size_t i = 0; i < N; i++) A[i] = psi_inv(A[i]);
    for (size_t i = 0; i < N; i++) {
        if ((A[i] >> 127) & 1) err = -1;          /* deg C_i <= 126 */
        if (i >= L && A[i] != 0) err = -2;         /* only L product blocks */
    }
    /* InterleavedCombine: out[w] = lo64(C_w) ^ hi64(C_(w-1)) */
    for (size_t w = 0; w < na + nb; w++) {
        uint64_t v = 0;
        if (w < N) v ^= (uint64_t)A[w];
        if (w >= 1 && w - 1 < N) v ^= (uint64_t)(A[w - 1] >> 64);
        c[w] = v;
    }
    free_constants(C, m);
    free(A); free(B);
    return err;
}

/* ------------------------------------------------------------------------------------------ */
/* O3, App. C: multiplication through the Frobenius bijection E_(beta_(m+64) + V_m) */
/*   "an FFT directly on GF(2)[x] ... abandoning the Kronecker segmentation".       */
/*   A binary polynomial of < 128 n bits (n = 2^m) is evaluated at the n points beta_(m+64) +    */
/*   phi(i), i < n (Def. P:1502-1507): BasisCvt on its 2^(m+7) GF(2) coefficients ("proceeded    */
/*   straightforwardly with alg. 3"), the first 7 layers of Alg. 1 with alpha =          */
/*   beta_(m+64) keeping block 0 only ("reserve only the first 1/128 results"; the   */
/*   "encoding"), then the normal n-point FFT_LCH with the same alpha.  The product */
/*   has < 128 n' bits for n' = the smallest power of two with 128 n' >= L (R23), so   */
/*   E(c) = E(a) E(b) pointwise is inverted by iFFT, decoding (the 128 x 128 map of the encoding */
/*   is invertible: Prop. P:1515-1518) and iBasisCvt.  The Cantor basis beta_i is the tower's    */
/*   v_i (phi(i) = i as a bit pattern), so alpha = 2^(m+64) and all arithmetic is TGF(2^128).    */
/* ------------------------------------------------------------------------------------------ */
/* Alg. 2/3 on GF(2) coefficients (one byte per bit): the same steps as taylor / cvt above */
static void taylor8(uint8_t *f, size_t s, size_t len, int K) {
    size_t h = len / 2, d = h - (h >> K);
    for (size_t i = len - 1; i >= h; i--) {
        f[s + i - d] ^= f[s + i];
        if (i == h) break;
    }
}
static void itaylor8(uint8_t *f, size_t s, size_t len, int K) {
    size_t h = len / 2, d = h - (h >> K);
    for (size_t i = h; i < len; i++) f[s + i - d] ^= f[s + i];
}
static void cvt8(uint8_t *f, size_t base, int m, int sigma) {
    if (m <= 1) return;
    int K = 1 << floor_log2(m - 1);
    for (int l = m; l >= K + 1; l--)
        for (size_t s = 0; s < ((size_t)1 << (m + sigma)); s += ((size_t)1 << (l + sigma)))
            taylor8(f, base + s, (size_t)1 << (l + sigma), K);
    cvt8(f, base, m - K, sigma + K);
    for (size_t c = 0; c < ((size_t)1 << (m + sigma)); c += ((size_t)1 << (K + sigma))) cvt8(f, base + c, K, sigma);
}
static void icvt8(uint8_t *f, size_t base, int m, int sigma) {
    if (m <= 1) return;
    int K = 1 << floor_log2(m - 1);
    for (size_t c = 0; c < ((size_t)1 << (m + sigma)); c += ((size_t)1 << (K + sigma))) icvt8(f, base + c, K, sigma);
    icvt8(f, base, m - K, sigma + K);
    for (int l = K + 1; l <= m; l++)
        for (size_t s = 0; s < ((size_t)1 << (m + sigma)); s += ((size_t)1 << (l + sigma)))
            itaylor8(f, base + s, (size_t)1 << (l + sigma), K);
}

/* BasisCvt / iBasisCvt on 2^M GF(2) coefficients packed little-endian in 2^(M-6) words (M >= 6), in place */
void or_basis_cvt_bits(uint64_t *words, int M, int inverse) {
    size_t NB = (size_t)1 << M;
    uint8_t *g = (uint8_t *)malloc(NB);
    for (size_t i = 0; i < NB; i++) g[i] = (words[i / 64] >> (i % 64)) & 1;
    if (inverse) icvt8(g, 0, M, 0); else cvt8(g, 0, M, 0);
    memset(words, 0, (NB / 64) * sizeof(uint64_t));
    for (size_t i = 0; i < NB; i++) if (g[i]) words[i / 64] |= (uint64_t)1 << (i % 64);
    free(g);
}

/* FFT_LCH / iFFT at displacement alpha: block b of layer k multiplies by s_k(alpha + phi(b)) =
 * s_k(alpha) + s_k(phi(b)) (s_k is linear) -- the alpha = 0 constants plus one per layer */
static void fft_alpha(u128 *A, int m, u128 **C, const u128 *sa, int inverse) {
    for (int kk = 0; kk < m; kk++) {
        int k = inverse ? kk : m - 1 - kk;
        size_t half = (size_t)1 << k, nb = (size_t)1 << (m - k - 1);
        for (size_t j = 0; j < nb; j++) {
            size_t b = j << (k + 1);
            u128 c = C[k][j] ^ sa[k];
            for (size_t i = 0; i < half; i++) {
                if (!inverse) {
                    A[b + i] ^= tmul(A[b + half + i], c, 7);
                    A[b + half + i] ^= A[b + i];
                } else {
                    A[b + half + i] ^= A[b + i];
                    A[b + i] ^= tmul(A[b + half + i], c, 7);
                }
            }
        }
    }
}

/* E_(alpha + V_m) of the 2^(m+7) novel-basis bits g: the first 7 layers of Alg. 1 (k = m+6 .. m) on
 * block 0 only -- A[i] ^= s_k(alpha) A[i + 2^k], i < 2^k (the upper half belongs to the points that are
 * not kept) -- then the n-point FFT with alpha.  stage 1: stop after the encoding. */
static void frob_eval(const uint8_t *g, int m, u128 alpha, u128 *E, int stage) {
    int M = m + 7;
    size_t NB = (size_t)1 << M, n = (size_t)1 << m;
    u128 *T = (u128 *)malloc(NB * sizeof(u128));
    for (size_t i = 0; i < NB; i++) T[i] = g[i];
    for (int k = M - 1; k >= m; k--) {
        u128 c = s_eval(k, alpha);
        for (size_t i = 0; i < ((size_t)1 << k); i++) T[i] ^= tmul(T[i + ((size_t)1 << k)], c, 7);
    }
    memcpy(E, T, n * sizeof(u128));
    free(T);
    if (stage == 1) return;
    u128 sa[64];
    for (int k = 0; k < m; k++) sa[k] = s_eval(k, alpha);
    u128 **C = all_constants(m);
    fft_alpha(E, m, C, sa, 0);
    free_constants(C, m);
}

/* Gauss-Jordan inverse of the 128 x 128 GF(2) matrix whose column j is col[j] (rows as u128 bit sets);
 * returns 0, or -1 if singular.  out[j] = column j of the inverse. */
static int gf2_inverse128(const u128 *col, u128 *out) {
    u128 rowA[128], rowI[128];
    for (int r = 0; r < 128; r++) {
        u128 v = 0;
        for (int j = 0; j < 128; j++) if ((col[j] >> r) & 1) v |= (u128)1 << j;
        rowA[r] = v; rowI[r] = (u128)1 << r;
    }
    for (int c = 0; c < 128; c++) {
        int p = -1;
        for (int r = c; r < 128; r++) if ((rowA[r] >> c) & 1) { p = r; break; }
        if (p < 0) return -1;
        u128 t = rowA[p]; rowA[p] = rowA[c]; rowA[c] = t;
        t = rowI[p]; rowI[p] = rowI[c]; rowI[c] = t;
        for (int r = 0; r < 128; r++)
            if (r != c && ((rowA[r] >> c) & 1)) { rowA[r] ^= rowA[c]; rowI[r] ^= rowI[c]; }
    }
    /* rowI[r] = row r of the inverse; column j = bits j of every row */
    for (int j = 0; j < 128; j++) {
        u128 v = 0;
        for (int r = 0; r < 128; r++) if ((rowI[r] >> j) & 1) v |= (u128)1 << r;
        out[j] = v;
    }
    return 0;
}
/* apply a matrix given by columns: y = sum_j x_j col[j] */
static u128 apply128(const u128 *col, u128 x) {
    u128 y = 0;
    for (int j = 0; j < 128; j++) if ((x >> j) & 1) y ^= col[j];
    return y;
}

/* the encoding's columns: the image of the unit bit j (g[i + j n] = 1) under the 7 layers */
static void frob_columns(int m, u128 alpha, u128 *col) {
    u128 sk[7];
    for (int b = 0; b < 7; b++) sk[b] = s_eval(m + b, alpha);
    for (int j = 0; j < 128; j++) {
        u128 c = 1;
        for (int b = 0; b < 7; b++) if ((j >> b) & 1) c = tmul(c, sk[b], 7);
        col[j] = c;
    }
}

static int frob_m(uint64_t L) { int m = 0; while (((uint64_t)128 << m) < L) m++; return m; }

/* E(a) at the 2^m points alpha + phi(i), alpha = beta_(m+64); a has a_bits <= 128 2^m bits.
 * out: 2^m tower elements (2 words each).  stage 1: the encoding only. */
int or_frob_eval(const uint64_t *a, uint64_t a_bits, int m, uint64_t *out, int stage) {
    tower_init();
    if (m < 0 || m > 40 || a_bits > ((uint64_t)128 << m)) return -1;
    int M = m + 7;
    size_t NB = (size_t)1 << M, n = (size_t)1 << m;
    uint8_t *g = (uint8_t *)calloc(NB, 1);
    for (uint64_t i = 0; i < a_bits; i++) g[i] = (a[i / 64] >> (i % 64)) & 1;
    cvt8(g, 0, M, 0);
    u128 *E = (u128 *)malloc(n * sizeof(u128));
    frob_eval(g, m, (u128)1 << (m + 64), E, stage);
    from128(E, n, 2, out);
    free(E); free(g);
    return 0;
}
/* the 128 columns of the encoding (2 words each), for the closed-form pin */
void or_frob_columns(int m, uint64_t *out) { tower_init(); u128 col[128]; frob_columns(m, (u128)1 << (m + 64), col); from128(col, 128, 2, out); }
int or_frob_m(uint64_t a_bits, uint64_t b_bits) { return a_bits && b_bits ? frob_m(a_bits + b_bits - 1) : 0; }

/* c = a b (na + nb words) through E: returns 0, or -1 (singular encoding), -2 (bits above the product) */
int or_frob_mul(const uint64_t *a, uint64_t a_bits, const uint64_t *b, uint64_t b_bits, uint64_t *c) {
    tower_init();
    size_t na = (a_bits + 63) / 64, nb = (b_bits + 63) / 64;
    memset(c, 0, (na + nb) * sizeof(uint64_t));
    if (a_bits == 0 || b_bits == 0) return 0;
    uint64_t L = a_bits + b_bits - 1;          /* coefficients of the product */
    int m = frob_m(L), M = m + 7;
    size_t NB = (size_t)1 << M, n = (size_t)1 << m;
    u128 alpha = (u128)1 << (m + 64);
    uint8_t *g = (uint8_t *)calloc(NB, 1);
    u128 *EA = (u128 *)malloc(n * sizeof(u128)), *EB = (u128 *)malloc(n * sizeof(u128));
    for (uint64_t i = 0; i < a_bits; i++) g[i] = (a[i / 64] >> (i % 64)) & 1;
    cvt8(g, 0, M, 0);
    frob_eval(g, m, alpha, EA, 2);
    memset(g, 0, NB);
    for (uint64_t i = 0; i < b_bits; i++) g[i] = (b[i / 64] >> (i % 64)) & 1;
    cvt8(g, 0, M, 0);
    frob_eval(g, m, alpha, EB, 2);
    /* E(c) = E(a) E(b) */
    for (size_t i = 0; i < n; i++) EA[i] = tmul(EA[i], EB[i], 7);
    /* iFFT with alpha */
    u128 sa[64];
    for (int k = 0; k < m; k++) sa[k] = s_eval(k, alpha);
    u128 **C = all_constants(m);
    fft_alpha(EA, m, C, sa, 1);
    free_constants(C, m);
    /* decoding: the 128 bits g[i + j n] of every i from the encoded element */
    u128 col[128], inv[128];
    frob_columns(m, alpha, col);
    int err = 0;
    if (gf2_inverse128(col, inv) != 0) err = -1;
    memset(g, 0, NB);
    for (size_t i = 0; i < n && !err; i++) {
        u128 bits = apply128(inv, EA[i]);
        for (int j = 0; j < 128; j++) g[i + (size_t)j * n] = (uint8_t)((bits >> j) & 1);
    }
    /* iBasisCvt on the 2^(m+7) GF(2) coefficients */
    icvt8(g, 0, M, 0);
    for (size_t i = 0; i < NB && !err; i++) {
        if (!g[i]) continue;
        if (i >= L) { err = -2; break; }
        c[i / 64] |= (uint64_t)1 << (i % 64);
    }
    free(g); free(EA); free(EB);
    return err;
}

/* ------------------------------------------------------------------------------------------ */
/* O3, Alg. 4 "simple" multiplication (sec 3.1): the working field stays GF(2^128) in    */
/* polynomial basis; FFT_LCH (Alg. 1) at the points psi^-1(phi_v(i)) with multipliers s_k computed */
/* in the Cantor (tower) basis "and then switched to its representation in GF(2^128) with a linear */
/* map": c = psi^-1(s_k(phi_v(b))), random-looking 128-bit elements.  No changeRepr.    */
/* ------------------------------------------------------------------------------------------ */
static void fft_poly(u128 *A, int m, u128 **C, int inverse) {
    for (int kk = 0; kk < m; kk++) {
        const int k = inverse ? kk : m - 1 - kk;
        size_t half = (size_t)1 << k, nb = (size_t)1 << (m - k - 1);
#pragma omp parallel for schedule(static) if (nb * half >= 4096)
        for (size_t j = 0; j < nb; j++) {
            size_t b = j << (k + 1);
            u128 c = psi_inv(C[k][j]);
            for (size_t i = 0; i < half; i++) {
                if (!inverse) {
                    A[b + i] ^= gf128_mul(A[b + half + i], c);
                    A[b + half + i] ^= A[b + i];
                } else {
                    A[b + half + i] ^= A[b + i];
                    A[b + i] ^= gf128_mul(A[b + half + i], c);
                }
            }
        }
    }
}
void or_fft_alg4(uint64_t *data, int m) {
    tower_init();
    psi_init();
    size_t n = (size_t)1 << m;
    u128 *A = (u128 *)malloc(n * sizeof(u128));
    u128 **C = all_constants(m);
    to128(data, n, 2, A); fft_poly(A, m, C, 0); from128(A, n, 2, data);
    free_constants(C, m); free(A);
}
/* Alg. 4 binPolyMul.  Stage dumps (optional, N x 2 words): after FFT_LCH (a), after pointmul. */
int or_alg4_mul(const uint64_t *a, uint64_t a_bits, const uint64_t *b, uint64_t b_bits, uint64_t *c,
                uint64_t *st_fft_a, uint64_t *st_prod) {
    tower_init();
    if (psi_init() != 0) return -10;
    size_t na = (a_bits + 63) / 64, nb = (b_bits + 63) / 64;
    if (a_bits == 0 || b_bits == 0) { memset(c, 0, (na + nb) * sizeof(uint64_t)); return 0; }
    size_t L = na + nb - 1;
    int m = ceil_log2_sz(L);
    size_t N = (size_t)1 << m;
    u128 *A = (u128 *)calloc(N, sizeof(u128)), *B = (u128 *)calloc(N, sizeof(u128));
    for (size_t j = 0; j < na; j++) {   /* Split */
        uint64_t w = a[j];
        if (j == na - 1 && (a_bits & 63)) w &= (((uint64_t)1) << (a_bits & 63)) - 1;
        A[j] = w;
    }
    for (size_t j = 0; j < nb; j++) {
        uint64_t w = b[j];
        if (j == nb - 1 && (b_bits & 63)) w &= (((uint64_t)1) << (b_bits & 63)) - 1;
        B[j] = w;
    }
    cvt(A, 0, m, 0); cvt(B, 0, m, 0);                       /* BasisCvt */
    u128 **C = all_constants(m);
    fft_poly(A, m, C, 0); fft_poly(B, m, C, 0);             /* FFT_LCH at phi_beta points */
    if (st_fft_a) from128(A, N, 2, st_fft_a);
#pragma omp parallel for schedule(static) if (N >= 4096)
    for (size_t i = 0; i < N; i++) A[i] = gf128_mul(A[i], B[i]);   /* pointmul in GF(2^128) */
    if (st_prod) from128(A, N, 2, st_prod);
    fft_poly(A, m, C, 1);                                   /* iFFT_LCH */
    icvt(A, 0, m, 0);                                       /* iBasisCvt */
    int err = 0;
    for (size_t i = 0; i < N; i++) {
        if ((A[i] >> 127) & 1) err = -1;
        if (i >= L && A[i] != 0) err = -2;
    }
    for (size_t w = 0; w < na + nb; w++) {                  /* InterleavedCombine */
        uint64_t v = 0;
        if (w < N) v ^= (uint64_t)A[w];
        if (w >= 1 && w - 1 < N) v ^= (uint64_t)(A[w - 1] >> 64);
        c[w] = v;
    }
    free_constants(C, m);
    free(A); free(B);
    return err;
}

/* ------------------------------------------------------------------------------------------ */
/* O3 w = 128: Alg. 5 with 128-bit blocks over TGF(2^256) ("An initial block width of w=128 bits */
/* is also possible and in this case the operative field is TGF(2^256)"; sec 4.2     */
/* P:1077-1114).                                                                                */
/*   TGF(2^256) = TGF(2^128)[x_8]/(x_8^2 + x_8 + P), P = x_1...x_7 = v_127: the tower definition */
/*    one level up; an element is (lo, hi) = lo + hi x_8 (bit k <-> v_k, k < 256).    */
/*   GF(2^256) in polynomial basis = GF(2)[z]/(z^256 + z^10 + z^5 + z^2 + 1) (R20: the  */
/*   paper names no degree-256 modulus; this pentanomial is irreducible, pinned by a Rabin test). */
/*   changeRepr_256 follows R9's rule: X_1^2+X_1 = 1, X_k^2+X_k = X_1...X_(k-1), k <= 8, each the */
/*   numerically smaller root; v_k -> prod_{bit j of k} X_(j+1).                                 */
/* ------------------------------------------------------------------------------------------ */
typedef struct { u128 lo, hi; } u256;
static inline u256 u256_xor(u256 a, u256 b) { u256 r = {a.lo ^ b.lo, a.hi ^ b.hi}; return r; }
static inline int u256_bit(u256 a, int i) { return (int)((i < 128 ? a.lo >> i : a.hi >> (i - 128)) & 1); }
static inline u256 u256_one(int i) {
    u256 r = {0, 0};
    if (i < 128) r.lo = ((u128)1) << i; else r.hi = ((u128)1) << (i - 128);
    return r;
}
static inline int u256_less(u256 a, u256 b) { return a.hi != b.hi ? a.hi < b.hi : a.lo < b.lo; }
static inline int u256_eq(u256 a, u256 b) { return a.hi == b.hi && a.lo == b.lo; }

/* Karatsuba at level 8 (sec 4.1.3): lo = a0b0 + a1b1 P, hi = (a0+a1)(b0+b1) + a0b0;
 * with one operand in TGF(2^128) it drops to two level-7 products (Prop. 2). */
static u256 tmul256(u256 a, u256 b) {
    u256 r;
    if (b.hi == 0) { r.lo = tmul(a.lo, b.lo, 7); r.hi = tmul(a.hi, b.lo, 7); return r; }
    if (a.hi == 0) { r.lo = tmul(a.lo, b.lo, 7); r.hi = tmul(a.lo, b.hi, 7); return r; }
    const u128 P = ((u128)1) << 127;   /* v_127 */
    u128 p0 = tmul(a.lo, b.lo, 7), p2 = tmul(a.hi, b.hi, 7), p1 = tmul(a.lo ^ a.hi, b.lo ^ b.hi, 7);
    r.lo = p0 ^ tmul(p2, P, 7);
    r.hi = p1 ^ p0;
    return r;
}
static inline u256 mk256(const uint64_t *w) { u256 r = {mk(w[0], w[1]), mk(w[2], w[3])}; return r; }
static inline void unmk256(u256 x, uint64_t *w) { unmk(x.lo, w); unmk(x.hi, w + 2); }
void or_tower256_mul(const uint64_t *a, const uint64_t *b, uint64_t *r) {
    tower_init();
    unmk256(tmul256(mk256(a), mk256(b)), r);
}

/* GF(2^256) polynomial basis: multiply by z modulo z^256 + z^10 + z^5 + z^2 + 1, shift-and-add */
static inline u256 gf256p_mulz(u256 a) {
    int carry = (int)(a.hi >> 127);
    a.hi = (a.hi << 1) | (a.lo >> 127);
    a.lo <<= 1;
    if (carry) a.lo ^= (u128)0x425;   /* z^10 + z^5 + z^2 + 1 */
    return a;
}
static u256 gf256p_mul(u256 a, u256 b) {
    u256 acc = {0, 0};
    for (int i = 0; i < 256; i++) {
        if (u256_bit(b, i)) acc = u256_xor(acc, a);
        a = gf256p_mulz(a);
    }
    return acc;
}
void or_gf256p_mul(const uint64_t *a, const uint64_t *b, uint64_t *r) { unmk256(gf256p_mul(mk256(a), mk256(b)), r); }

/* Gauss-Jordan on a 256 x 256 GF(2) system given by the images col[i] of the unit vectors:
 * solves M x = c (returns 0 and the solution with free variables 0, or -1), used for the
 * Artin-Schreier equations r^2 + r = c (kernel {0, 1}) and for inverting changeRepr_256. */
static int solve256(const u256 *col, u256 c, u256 *x_out) {
    static u256 row[256]; static int rhs[256], pivcol[256];
    for (int r = 0; r < 256; r++) {
        u256 v = {0, 0};
        for (int i = 0; i < 256; i++) if (u256_bit(col[i], r)) v = u256_xor(v, u256_one(i));
        row[r] = v; rhs[r] = u256_bit(c, r);
    }
    int nr = 0;
    for (int cidx = 0; cidx < 256 && nr < 256; cidx++) {
        int p = -1;
        for (int r = nr; r < 256; r++) if (u256_bit(row[r], cidx)) { p = r; break; }
        if (p < 0) continue;
        u256 t = row[p]; row[p] = row[nr]; row[nr] = t;
        int tr = rhs[p]; rhs[p] = rhs[nr]; rhs[nr] = tr;
        for (int r = 0; r < 256; r++)
            if (r != nr && u256_bit(row[r], cidx)) { row[r] = u256_xor(row[r], row[nr]); rhs[r] ^= rhs[nr]; }
        pivcol[nr] = cidx; nr++;
    }
    for (int r = nr; r < 256; r++) if (rhs[r]) return -1;
    u256 x = {0, 0};
    for (int r = 0; r < nr; r++) if (rhs[r]) x = u256_xor(x, u256_one(pivcol[r]));
    *x_out = x;
    return 0;
}

static u256 g_Mcol256[256], g_psicol256[256], g_X256[9];
static int g_psi256_ready = 0;
static int psi256_init(void) {
    if (g_psi256_ready) return 0;
    static u256 asc[256];   /* L(x) = x^2 + x on the unit vectors */
    for (int i = 0; i < 256; i++) { u256 e = u256_one(i); asc[i] = u256_xor(gf256p_mul(e, e), e); }
    u256 prod = u256_one(0);
    for (int k = 1; k <= 8; k++) {
        u256 r;
        if (solve256(asc, prod, &r) != 0) return -1;
        u256 alt = u256_xor(r, u256_one(0));   /* the other root */
        g_X256[k] = u256_less(alt, r) ? alt : r;
        prod = gf256p_mul(prod, g_X256[k]);
    }
    for (int k = 0; k < 256; k++) {
        u256 v = u256_one(0);
        for (int j = 0; j < 8; j++) if ((k >> j) & 1) v = gf256p_mul(v, g_X256[j + 1]);
        g_Mcol256[k] = v;
    }
    /* psi_256 = Mcol^-1: column c = the solution of M x = e_c */
    for (int c = 0; c < 256; c++)
        if (solve256(g_Mcol256, u256_one(c), &g_psicol256[c]) != 0) return -2;
    g_psi256_ready = 1;
    return 0;
}
static u256 apply_cols256(const u256 *cols, u256 x) {
    u256 r = {0, 0};
    for (int i = 0; i < 256; i++) if (u256_bit(x, i)) r = u256_xor(r, cols[i]);
    return r;
}
static inline u256 psi256(u256 x) { return apply_cols256(g_psicol256, x); }      /* poly -> tower */
static inline u256 psi256_inv(u256 x) { return apply_cols256(g_Mcol256, x); }   /* tower -> poly */
int or_psi256_init(void) { return psi256_init(); }
void or_psi256(const uint64_t *x, uint64_t *r) { psi256_init(); unmk256(psi256(mk256(x)), r); }
void or_psi256_inv(const uint64_t *x, uint64_t *r) { psi256_init(); unmk256(psi256_inv(mk256(x)), r); }
void or_psi256_generator(int k, uint64_t *r) { psi256_init(); unmk256(g_X256[k], r); }

/* FFT_LCH / iFFT_LCH (Alg. 1) on TGF(2^256) elements; the multipliers are the
 * same s_k(phi_v(b)) as at w = 64 (they lie in the subfield spanned by v_0..v_(m-1)). */
static void fft256(u256 *A, int m, u128 **C) {
    for (int k = m - 1; k >= 0; k--) {
        size_t half = (size_t)1 << k, nb = (size_t)1 << (m - k - 1);
#pragma omp parallel for schedule(static) if (nb * half >= 4096)
        for (size_t j = 0; j < nb; j++) {
            size_t b = j << (k + 1);
            u256 c = {C[k][j], 0};
            for (size_t i = 0; i < half; i++) {
                A[b + i] = u256_xor(A[b + i], tmul256(A[b + half + i], c));
                A[b + half + i] = u256_xor(A[b + half + i], A[b + i]);
            }
        }
    }
}
static void ifft256(u256 *A, int m, u128 **C) {
    for (int k = 0; k < m; k++) {
        size_t half = (size_t)1 << k, nb = (size_t)1 << (m - k - 1);
#pragma omp parallel for schedule(static) if (nb * half >= 4096)
        for (size_t j = 0; j < nb; j++) {
            size_t b = j << (k + 1);
            u256 c = {C[k][j], 0};
            for (size_t i = 0; i < half; i++) {
                A[b + half + i] = u256_xor(A[b + half + i], A[b + i]);
                A[b + i] = u256_xor(A[b + i], tmul256(A[b + half + i], c));
            }
        }
    }
}
void or_fft256(uint64_t *data, int m) {
    tower_init();
    size_t n = (size_t)1 << m;
    u256 *A = (u256 *)malloc(n * sizeof(u256));
    u128 **C = all_constants(m);
    for (size_t i = 0; i < n; i++) A[i] = mk256(data + 4 * i);
    fft256(A, m, C);
    for (size_t i = 0; i < n; i++) unmk256(A[i], data + 4 * i);
    free_constants(C, m); free(A);
}

/* Alg. 5 with w = 128.  Stage dumps (optional, N x 4 words, tower elements): after changeRepr,
 * after FFT_LCH (a), after pointmul, after iBasisCvt.  c receives na+nb 64-bit words. */
int or_alg5_mul_w128(const uint64_t *a, uint64_t a_bits, const uint64_t *b, uint64_t b_bits, uint64_t *c,
                     uint64_t *st_cvt_a, uint64_t *st_fft_a, uint64_t *st_prod, uint64_t *st_icvt) {
    tower_init();
    if (psi256_init() != 0) return -10;
    size_t na = (a_bits + 63) / 64, nb = (b_bits + 63) / 64;
    if (a_bits == 0 || b_bits == 0) { memset(c, 0, (na + nb) * sizeof(uint64_t)); return 0; }
    size_t ma = (a_bits + 127) / 128, mb = (b_bits + 127) / 128;   /* 128-bit blocks */
    size_t L = ma + mb - 1;
    int m = ceil_log2_sz(L);
    size_t N = (size_t)1 << m;
    u128 *Fa = (u128 *)calloc(N, sizeof(u128)), *Fb = (u128 *)calloc(N, sizeof(u128));
    /* Split into 128-bit blocks (w = 128): block j = words 2j, 2j+1; bits >= a_bits masked */
    for (uint64_t i = 0; i < a_bits; i++) if ((a[i >> 6] >> (i & 63)) & 1) Fa[i >> 7] |= ((u128)1) << (i & 127);
    for (uint64_t i = 0; i < b_bits; i++) if ((b[i >> 6] >> (i & 63)) & 1) Fb[i >> 7] |= ((u128)1) << (i & 127);
    /* BasisCvt on the 128-bit blocks (XOR-only on whole blocks) */
    cvt(Fa, 0, m, 0); cvt(Fb, 0, m, 0);
    /* changeRepr into TGF(2^256): the block is an element of degree < 128 */
    u256 *A = (u256 *)malloc(N * sizeof(u256)), *B = (u256 *)malloc(N * sizeof(u256));
#pragma omp parallel for schedule(static) if (N >= 4096)
    for (size_t i = 0; i < N; i++) {
        u256 xa = {Fa[i], 0}, xb = {Fb[i], 0};
        A[i] = psi256(xa); B[i] = psi256(xb);
    }
    free(Fa); free(Fb);
    if (st_cvt_a) for (size_t i = 0; i < N; i++) unmk256(A[i], st_cvt_a + 4 * i);
    u128 **C = all_constants(m);
    fft256(A, m, C); fft256(B, m, C);
    if (st_fft_a) for (size_t i = 0; i < N; i++) unmk256(A[i], st_fft_a + 4 * i);
#pragma omp parallel for schedule(static) if (N >= 4096)
    for (size_t i = 0; i < N; i++) A[i] = tmul256(A[i], B[i]);   /* pointmul P:898-899 */
    if (st_prod) for (size_t i = 0; i < N; i++) unmk256(A[i], st_prod + 4 * i);
    ifft256(A, m, C);
    /* iBasisCvt in the tower representation: XOR-only on whole 256-bit units, i.e. the
     * same network applied to the low and the high 128-bit halves */
    u128 *Lo = (u128 *)malloc(N * sizeof(u128)), *Hi = (u128 *)malloc(N * sizeof(u128));
    for (size_t i = 0; i < N; i++) { Lo[i] = A[i].lo; Hi[i] = A[i].hi; }
    icvt(Lo, 0, m, 0); icvt(Hi, 0, m, 0);
    for (size_t i = 0; i < N; i++) { A[i].lo = Lo[i]; A[i].hi = Hi[i]; }
    free(Lo); free(Hi);
    if (st_icvt) for (size_t i = 0; i < N; i++) unmk256(A[i], st_icvt + 4 * i);
    /* changeRepr back */
    int err = 0;
#pragma omp parallel for schedule(static) if (N >= 4096)
    for (size_t i = 0; i < N; i++) A[i] = psi256_inv(A[i]);
    for (size_t i = 0; i < N; i++) {
        if ((A[i].hi >> 127) & 1) err = -1;                        /* deg C_i <= 254 */
        if (i >= L && (A[i].lo | A[i].hi) != 0) err = -2;
    }
    /* InterleavedCombine on 128-bit blocks: out[w] = lo128(C_w) ^ hi128(C_(w-1)) */
    for (size_t w = 0; w < na + nb; w++) {
        size_t blk = w >> 1;
        u128 v = 0;
        if (blk < N) v ^= A[blk].lo;
        if (blk >= 1 && blk - 1 < N) v ^= A[blk - 1].hi;
        c[w] = (w & 1) ? (uint64_t)(v >> 64) : (uint64_t)v;
    }
    free_constants(C, m);
    free(A); free(B);
    return err;
}

/* ------------------------------------------------------------------------------------------ */
/* O4: product check modulo random irreducible degree-64 polynomials (SURVEY c.2 O4)            */
/*   p = x^64 + r(x); x^64 == r (mod p).                                                        */
/* ------------------------------------------------------------------------------------------ */
static uint64_t mulmod64(uint64_t x, uint64_t y, uint64_t r) {
    u128 t = clmul64(x, y);
    uint64_t hi = (uint64_t)(t >> 64), lo = (uint64_t)t;
    /* t = hi x^64 + lo == hi r + lo; hi r has degree < 127; fold twice */
    while (hi) {
        u128 u = clmul64(hi, r);
        lo ^= (uint64_t)u;
        hi = (uint64_t)(u >> 64);
    }
    return lo;
}
/* polynomial gcd over GF(2) of a (deg <= 64, as u128) and p */
static int deg128(u128 x) { int d = -1; while (x) { d++; x >>= 1; } return d; }
static u128 pgcd(u128 a, u128 b) {
    while (b) {
        while (a && deg128(a) >= deg128(b)) a ^= b << (deg128(a) - deg128(b));
        u128 t = a; a = b; b = t;
    }
    return a;
}
/* Rabin test for degree 64: x^(2^64) == x mod p, gcd(x^(2^32) - x, p) = 1. */
int or_is_irreducible64(uint64_t r) {
    clmul_init();
    if (!(r & 1)) return 0;
    uint64_t x = 2, t = x;
    uint64_t t32 = 0;
    for (int i = 0; i < 64; i++) { t = mulmod64(t, t, r); if (i == 31) t32 = t; }
    if (t != x) return 0;
    u128 p = ((u128)1 << 64) | r;
    u128 g = pgcd((u128)(t32 ^ x), p);
    return deg128(g) == 0;
}
/* residue of a polynomial of n words modulo p (Horner from the top word: r <- r x^64 + w) */
uint64_t or_poly_mod(const uint64_t *a, size_t n, uint64_t r) {
    clmul_init();
    uint64_t acc = 0;
    for (size_t i = n; i-- > 0;) acc = mulmod64(acc, r, r) ^ a[i];
    return acc;
}
uint64_t or_mulmod64(uint64_t x, uint64_t y, uint64_t r) { clmul_init(); return mulmod64(x, y, r); }

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
void or_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
