// field_host.h -- host-side field arithmetic and constant-table construction for the CUDA path.
//
// Product-side code: written independently of oracle/ (which the product never links).  The tower
// product here is computed by the "basis expansion" route -- a * b = XOR over set bits j of b of
// a * v_j, with a * v_j obtained by multiplying by the generators x_i (SWAR on 2^i-bit blocks) --
// rather than the oracle's Karatsuba recursion.
//
// Tower (§3.2): TGF(2^(2^i)) = TGF(2^(2^(i-1)))[x_i]/(x_i^2 + x_i + P_(i-1)),
// P_(i-1) = x_1 ... x_(i-1) (P_0 = 1).  Element bit k = coordinate of v_k (Def. v_k).
#pragma once
#include <stdint.h>
#include <string.h>
#include <utility>

namespace gf2x_host {

typedef unsigned __int128 u128;

static inline u128 lowmask_blocks(int i) {
    // mask selecting the low half of every 2^i-bit block (1 <= i <= 7)
    if (i < 1 || i > 7) return 0;
    int h = 1 << (i - 1);
    u128 m = 0;
    for (int blk = 0; blk < 128; blk += (1 << i)) m |= ((((u128)1) << h) - 1) << blk;
    return m;
}

u128 mul_P(u128 x, int i);

// multiply every 2^i-bit block of x (a TGF(2^(2^i)) element) by the generator x_i:
// (u0 + u1 x_i) x_i = P_(i-1) u1 + (u0 + u1) x_i
static inline u128 mul_gen(u128 x, int i) {
    if (i < 1 || i > 7) return 0;
    int h = 1 << (i - 1);
    u128 lo = lowmask_blocks(i);
    u128 u0 = x & lo, u1 = (x >> h) & lo;
    return mul_P(u1, i - 1) | ((u0 ^ u1) << h);
}

// multiply every 2^i-bit block by P_i = x_1 ... x_i (P_0 = 1)
inline u128 mul_P(u128 x, int i) {
    for (int g = 1; g <= i; g++) x = mul_gen(x, g);
    return x;
}

// a * v_j (j < 128): v_j = prod_{bit t of j} x_(t+1)
static inline u128 mul_basis(u128 a, int j) {
    for (int t = 0; t < 7; t++)
        if ((j >> t) & 1) a = mul_gen(a, t + 1);
    return a;
}

// general tower product (both operands in TGF(2^128))
static inline u128 tower_mul(u128 a, u128 b) {
    u128 acc = 0;
    for (int j = 0; j < 128; j++)
        if ((b >> j) & 1) acc ^= mul_basis(a, j);
    return acc;
}

// s_1(x) = x^2 + x ; s_k = s_1 iterated k times (corollary P:718-721)
static inline u128 s1(u128 x) { return tower_mul(x, x) ^ x; }

// ----------------------------------------------------------- GF(2^128) polynomial basis
// GF(2)[z]/(z^128 + z^7 + z^2 + z + 1)  (§2.2.1)
static inline u128 gf128_mul(u128 a, u128 b) {
    u128 r = 0;
    while (b) {
        if (b & 1) r ^= a;
        b >>= 1;
        u128 top = a >> 127;
        a <<= 1;
        if (top) a ^= 0x87;
    }
    return r;
}

// Solve y^2 + y = c (kernel {0,1}) by elimination; returns the numerically smaller root.
// Returns false if c has trace 1 (no solution).
static inline bool gf128_artin_schreier(u128 c, u128* out) {
    // rows r: equation for output bit r; columns: unknown bits.  Column j image = z^(2j) + z^j.
    u128 img[128];
    for (int j = 0; j < 128; j++) {
        u128 e = ((u128)1) << j;
        img[j] = gf128_mul(e, e) ^ e;
    }
    // build augmented rows as (coefficient row, rhs bit)
    u128 row[128];
    unsigned char rhs[128];
    for (int r = 0; r < 128; r++) {
        u128 v = 0;
        for (int j = 0; j < 128; j++) v |= ((img[j] >> r) & 1) << j;
        row[r] = v;
        rhs[r] = (unsigned char)((c >> r) & 1);
    }
    int where[128];
    for (int j = 0; j < 128; j++) where[j] = -1;
    int r = 0;
    for (int j = 0; j < 128 && r < 128; j++) {
        int p = -1;
        for (int i = r; i < 128; i++)
            if ((row[i] >> j) & 1) { p = i; break; }
        if (p < 0) continue;
        u128 t = row[p]; row[p] = row[r]; row[r] = t;
        unsigned char tb = rhs[p]; rhs[p] = rhs[r]; rhs[r] = tb;
        for (int i = 0; i < 128; i++)
            if (i != r && ((row[i] >> j) & 1)) { row[i] ^= row[r]; rhs[i] ^= rhs[r]; }
        where[j] = r++;
    }
    for (int i = r; i < 128; i++)
        if (rhs[i]) return false;
    u128 y = 0;
    for (int j = 0; j < 128; j++)
        if (where[j] >= 0 && rhs[where[j]]) y |= ((u128)1) << j;
    u128 y2 = y ^ 1;
    *out = y < y2 ? y : y2;
    return true;
}

// changeRepr (§4.3) under DESIGN.md reading R9: images X_k of the generators x_k with
// X_1^2+X_1 = 1, X_k^2+X_k = X_1...X_(k-1), each the numerically smaller root; tower basis v_j maps
// to prod_{bit t of j} X_(t+1).  towerToPoly[j] = image of v_j; polyToTower[i] = image of z^i.
struct Isomorphism {
    u128 towerToPoly[128];
    u128 polyToTower[128];
    bool ok;
};

static inline Isomorphism build_isomorphism() {
    Isomorphism iso;
    iso.ok = false;
    u128 X[8];
    u128 prod = 1;
    for (int k = 1; k <= 7; k++) {
        if (!gf128_artin_schreier(prod, &X[k])) return iso;
        prod = gf128_mul(prod, X[k]);
    }
    for (int j = 0; j < 128; j++) {
        u128 v = 1;
        for (int t = 0; t < 7; t++)
            if ((j >> t) & 1) v = gf128_mul(v, X[t + 1]);
        iso.towerToPoly[j] = v;
    }
    // invert: solve M y = z^i for each i via elimination on [M | I] stored row-wise
    u128 A[128], B[128];
    for (int r = 0; r < 128; r++) {
        u128 v = 0;
        for (int j = 0; j < 128; j++) v |= ((iso.towerToPoly[j] >> r) & 1) << j;
        A[r] = v;
        B[r] = ((u128)1) << r;
    }
    for (int j = 0; j < 128; j++) {
        int p = -1;
        for (int i = j; i < 128; i++)
            if ((A[i] >> j) & 1) { p = i; break; }
        if (p < 0) return iso;
        u128 t = A[p]; A[p] = A[j]; A[j] = t;
        t = B[p]; B[p] = B[j]; B[j] = t;
        for (int i = 0; i < 128; i++)
            if (i != j && ((A[i] >> j) & 1)) { A[i] ^= A[j]; B[i] ^= B[j]; }
    }
    // row j of M^-1 is B[j]; column i of M^-1 (image of z^i) has bit j = bit i of B[j]
    for (int i = 0; i < 128; i++) {
        u128 v = 0;
        for (int j = 0; j < 128; j++) v |= ((B[j] >> i) & 1) << j;
        iso.polyToTower[i] = v;
    }
    iso.ok = true;
    return iso;
}


// ----------------------------------------------------------- w = 128: GF(2^256) and changeRepr_256
// GF(2)[z]/(z^256 + z^10 + z^5 + z^2 + 1) (R20), elements as 4 little-endian words.  The
// w = 128 variant embeds 128-bit blocks here and maps them to TGF(2^256) =
// TGF(2^128)[x_8]/(x_8^2 + x_8 + v_127) by the R9 rule one level up.
struct W256 {
    uint64_t w[4];
};
static inline W256 w256_zero() { W256 r; memset(&r, 0, sizeof(r)); return r; }
static inline W256 w256_unit(int i) { W256 r = w256_zero(); r.w[i >> 6] = 1ull << (i & 63); return r; }
static inline int w256_bit(const W256& a, int i) { return (int)((a.w[i >> 6] >> (i & 63)) & 1); }
static inline void w256_xor(W256& a, const W256& b) { for (int i = 0; i < 4; i++) a.w[i] ^= b.w[i]; }
static inline bool w256_less(const W256& a, const W256& b) {
    for (int i = 3; i >= 0; i--) if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
    return false;
}

// a * b: schoolbook over 64-bit digits into 8 words, then reduction of words 4..7 by the modulus
static inline W256 gf256p_mul(const W256& a, const W256& b) {
    uint64_t t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++)
            for (int k = 0; k < 64; k++)
                if ((b.w[j] >> k) & 1) {   // a.w[i] * z^(64 (i+j) + k)
                    const int sh = k, dst = i + j;
                    t[dst] ^= a.w[i] << sh;
                    if (sh) t[dst + 1] ^= a.w[i] >> (64 - sh);
                }
    // z^256 = z^10 + z^5 + z^2 + 1: fold bits >= 256 from the top down
    for (int bit = 511; bit >= 256; bit--)
        if ((t[bit >> 6] >> (bit & 63)) & 1) {
            t[bit >> 6] ^= 1ull << (bit & 63);
            const int base = bit - 256;
            const int offs[4] = {0, 2, 5, 10};
            for (int o : offs) t[(base + o) >> 6] ^= 1ull << ((base + o) & 63);
        }
    W256 r;
    for (int i = 0; i < 4; i++) r.w[i] = t[i];
    return r;
}

// Solve M x = c over GF(2), M given by the images of the 256 unit vectors (Gauss-Jordan; free
// variables 0).  Returns false if inconsistent.
static inline bool w256_solve(const W256* img, const W256& c, W256* x) {
    static W256 row[256];
    static unsigned char rhs[256];
    for (int r = 0; r < 256; r++) {
        row[r] = w256_zero();
        for (int j = 0; j < 256; j++)
            if (w256_bit(img[j], r)) row[r].w[j >> 6] |= 1ull << (j & 63);
        rhs[r] = (unsigned char)w256_bit(c, r);
    }
    int where[256];
    for (int j = 0; j < 256; j++) where[j] = -1;
    int r = 0;
    for (int j = 0; j < 256 && r < 256; j++) {
        int p = -1;
        for (int i = r; i < 256; i++)
            if (w256_bit(row[i], j)) { p = i; break; }
        if (p < 0) continue;
        std::swap(row[p], row[r]);
        std::swap(rhs[p], rhs[r]);
        for (int i = 0; i < 256; i++)
            if (i != r && w256_bit(row[i], j)) { w256_xor(row[i], row[r]); rhs[i] ^= rhs[r]; }
        where[j] = r++;
    }
    for (int i = r; i < 256; i++)
        if (rhs[i]) return false;
    *x = w256_zero();
    for (int j = 0; j < 256; j++)
        if (where[j] >= 0 && rhs[where[j]]) x->w[j >> 6] |= 1ull << (j & 63);
    return true;
}

// towerToPoly[j] = image of tower basis v_j (j < 256), polyToTower[i] = image of z^i
struct Isomorphism256 {
    W256 towerToPoly[256];
    W256 polyToTower[256];
    bool ok;
};
static inline bool build_isomorphism256(Isomorphism256* iso) {
    iso->ok = false;
    static W256 as_img[256];
    for (int j = 0; j < 256; j++) {
        W256 e = w256_unit(j);
        as_img[j] = gf256p_mul(e, e);
        w256_xor(as_img[j], e);
    }
    W256 X[9];
    W256 prod = w256_unit(0);
    for (int k = 1; k <= 8; k++) {
        W256 y;
        if (!w256_solve(as_img, prod, &y)) return false;
        W256 y2 = y;
        y2.w[0] ^= 1;
        X[k] = w256_less(y2, y) ? y2 : y;
        prod = gf256p_mul(prod, X[k]);
    }
    for (int j = 0; j < 256; j++) {
        W256 v = w256_unit(0);
        for (int t = 0; t < 8; t++)
            if ((j >> t) & 1) v = gf256p_mul(v, X[t + 1]);
        iso->towerToPoly[j] = v;
    }
    for (int i = 0; i < 256; i++)
        if (!w256_solve(iso->towerToPoly, w256_unit(i), &iso->polyToTower[i])) return false;
    iso->ok = true;
    return true;
}

}  // namespace gf2x_host
