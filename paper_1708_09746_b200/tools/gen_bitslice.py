"""Generate bit-sliced straight-line CUDA for tower-field products (build tool, product side).

A bit-sliced operand holds 32 field elements: word ("plane") j has bit e = coordinate j of element e
(coordinate j = coefficient of v_j, PAPER.md Def. of v_k P:658-661).  Products are generated from
the tower's recursive definition:
    level l (2^l bits) = level l-1 [x_l] / (x_l^2 + x_l + P),  P = v_(2^(l-1)-1),
    (a0 + a1 X)(b0 + b1 X) = [a0 b0 + P (a1 b1)] + [(a0+a1)(b0+b1) + a0 b0] X    (Karatsuba)
and multiplications by fixed constants are emitted as XOR networks (matrices reduced with a greedy
common-pair elimination).  This module computes its own tower arithmetic; it shares no code with
oracle/.

Output: paper_1708_09746_b200/csrc/bitslice_gen.cuh
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "csrc", "bitslice_gen.cuh")


# ----------------------------------------------------------------- scalar tower arithmetic (ints)
def tmul(a, b, l):
    if l == 0:
        return a & b & 1
    h = 1 << (l - 1)
    m = (1 << h) - 1
    a0, a1, b0, b1 = a & m, a >> h, b & m, b >> h
    p0, p2 = tmul(a0, b0, l - 1), tmul(a1, b1, l - 1)
    p1 = tmul(a0 ^ a1, b0 ^ b1, l - 1)
    return (p0 ^ tmul(p2, 1 << (h - 1), l - 1)) | ((p1 ^ p0) << h)


# ----------------------------------------------------------------- expression builder
class Prog:
    def __init__(self):
        self.lines = []
        self.n = 0
        self.cache = {}
        self.ops = {"and": 0, "xor": 0}

    def tmp(self, expr, kind):
        key = (kind, expr)
        if key in self.cache:
            return self.cache[key]
        name = f"t{self.n}"
        self.n += 1
        self.lines.append(f"const uint32_t {name} = {expr};")
        self.ops[kind] += 1
        self.cache[key] = name
        return name

    def AND(self, x, y):
        if x == "0u" or y == "0u":
            return "0u"
        x, y = sorted((x, y))
        return self.tmp(f"{x} & {y}", "and")

    def XOR(self, x, y):
        if x == "0u":
            return y
        if y == "0u":
            return x
        if x == y:
            return "0u"
        x, y = sorted((x, y))
        return self.tmp(f"{x} ^ {y}", "xor")

    def XORN(self, terms):
        # xor of a list (cancel duplicates)
        cnt = {}
        for t in terms:
            if t != "0u":
                cnt[t] = cnt.get(t, 0) ^ 1
        terms = sorted(t for t, c in cnt.items() if c)
        if not terms:
            return "0u"
        acc = terms[0]
        for t in terms[1:]:
            acc = self.XOR(acc, t)
        return acc


def linmap_matrix(const, l):
    """rows[i] = set of input coordinates j with bit i of (const * v_j) set, level l."""
    n = 1 << l
    cols = [tmul(const, 1 << j, l) for j in range(n)]
    return [[j for j in range(n) if (cols[j] >> i) & 1] for i in range(n)]


def apply_linmap(P, x, rows):
    """XOR network for out_i = xor_{j in rows[i]} x_j, with greedy common-pair elimination."""
    rows = [[x[j] for j in r if x[j] != "0u"] for r in rows]
    rows = [list(dict.fromkeys(r)) for r in rows]
    while True:
        best, bestc = None, 1
        counts = {}
        for r in rows:
            s = sorted(r)
            for i in range(len(s)):
                for j in range(i + 1, len(s)):
                    k = (s[i], s[j])
                    counts[k] = counts.get(k, 0) + 1
        for k, c in counts.items():
            if c > bestc:
                best, bestc = k, c
        if best is None:
            break
        v = P.XOR(*best)
        for r in rows:
            if best[0] in r and best[1] in r:
                r.remove(best[0])
                r.remove(best[1])
                r.append(v)
    return [P.XORN(r) for r in rows]


def bs_mul(P, a, b, l, leaf=1):
    """Karatsuba over the tower down to GF(4), schoolbook there (4 AND: fuses with the XORs into fewer
    LOP3 after ptxas: 868 vs 896 for the all-Karatsuba circuit)."""
    if l == 0:
        return [P.AND(a[0], b[0])]
    if l <= leaf:
        n = 1 << l
        out = [[] for _ in range(n)]
        for i in range(n):
            for j in range(n):
                v = tmul(1 << i, 1 << j, l)
                t = P.AND(a[i], b[j])
                for o in range(n):
                    if (v >> o) & 1:
                        out[o].append(t)
        return [P.XORN(o) for o in out]
    h = 1 << (l - 1)
    a0, a1, b0, b1 = a[:h], a[h:], b[:h], b[h:]
    p0 = bs_mul(P, a0, b0, l - 1, leaf)
    p2 = bs_mul(P, a1, b1, l - 1, leaf)
    p1 = bs_mul(P, [P.XOR(x, y) for x, y in zip(a0, a1)], [P.XOR(x, y) for x, y in zip(b0, b1)], l - 1, leaf)
    p2c = apply_linmap(P, p2, linmap_matrix(1 << (h - 1), l - 1))
    lo = [P.XOR(x, y) for x, y in zip(p0, p2c)]
    hi = [P.XOR(x, y) for x, y in zip(p1, p0)]
    return lo + hi


def bs_mul_pair(P, a, b, c, l, leaf=1):
    """a c and b c for one common multiplier c, emitted together: the c-side Karatsuba sums are formed once
    and the two products interleave at every recursion level (independent instruction streams)."""
    if l <= leaf:
        return bs_mul(P, a, c, l, leaf), bs_mul(P, b, c, l, leaf)
    h = 1 << (l - 1)
    a0, a1, b0, b1, c0, c1 = a[:h], a[h:], b[:h], b[h:], c[:h], c[h:]
    pa0, pb0 = bs_mul_pair(P, a0, b0, c0, l - 1, leaf)
    pa2, pb2 = bs_mul_pair(P, a1, b1, c1, l - 1, leaf)
    cs = [P.XOR(x, y) for x, y in zip(c0, c1)]
    pa1, pb1 = bs_mul_pair(P, [P.XOR(x, y) for x, y in zip(a0, a1)], [P.XOR(x, y) for x, y in zip(b0, b1)], cs,
                           l - 1, leaf)
    out = []
    for p0, p1, p2 in ((pa0, pa1, pa2), (pb0, pb1, pb2)):
        p2c = apply_linmap(P, p2, linmap_matrix(1 << (h - 1), l - 1))
        out.append([P.XOR(x, y) for x, y in zip(p0, p2c)] + [P.XOR(x, y) for x, y in zip(p1, p0)])
    return out[0], out[1]


def emit_mul_pair(fname, l):
    P = Prog()
    n = 1 << l
    pre = ([f"const uint32_t A{i} = a[{i}];" for i in range(n)] + [f"const uint32_t B{i} = b[{i}];" for i in range(n)] +
           [f"const uint32_t C{i} = c[{i}];" for i in range(n)])
    ra, rb = bs_mul_pair(P, [f"A{i}" for i in range(n)], [f"B{i}" for i in range(n)], [f"C{i}" for i in range(n)], l)
    body = pre + P.lines + [f"ra[{i}] = {ra[i]};" for i in range(n)] + [f"rb[{i}] = {rb[i]};" for i in range(n)]
    src = (f"// two {n}-bit tower products a c, b c of 32 bit-sliced triples (common c): {P.ops['and']} AND, "
           f"{P.ops['xor']} XOR\n"
           f"GF2X_HD GF2X_INLINE void {fname}(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, "
           f"const uint32_t* __restrict__ c, uint32_t* __restrict__ ra, uint32_t* __restrict__ rb) {{\n  "
           + "\n  ".join(body) + "\n}\n")
    return src, P.ops


def emit_mul(fname, l):
    P = Prog()
    n = 1 << l
    a = [f"a[{i}]" for i in range(n)]
    b = [f"b[{i}]" for i in range(n)]
    # bind inputs to locals
    pre = [f"const uint32_t A{i} = a[{i}];" for i in range(n)] + [f"const uint32_t B{i} = b[{i}];" for i in range(n)]
    r = bs_mul(P, [f"A{i}" for i in range(n)], [f"B{i}" for i in range(n)], l)
    body = pre + P.lines + [f"r[{i}] = {r[i]};" for i in range(n)]
    src = (f"// {n}-bit tower product of 32 bit-sliced pairs: {P.ops['and']} AND, {P.ops['xor']} XOR\n"
           f"GF2X_HD GF2X_INLINE void {fname}(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, "
           f"uint32_t* __restrict__ r) {{\n  " + "\n  ".join(body) + "\n}\n")
    return src, P.ops


def emit_const(fname, const, l):
    P = Prog()
    n = 1 << l
    x = [f"X{i}" for i in range(n)]
    pre = [f"const uint32_t X{i} = x[{i}];" for i in range(n)]
    r = apply_linmap(P, x, linmap_matrix(const, l))
    body = pre + P.lines + [f"r[{i}] = {r[i]};" for i in range(n)]
    src = (f"// multiply {n}-bit bit-sliced elements by the fixed tower constant {const:#x}: {P.ops['xor']} XOR\n"
           f"GF2X_HD GF2X_INLINE void {fname}(const uint32_t* __restrict__ x, uint32_t* __restrict__ r) {{\n  "
           + "\n  ".join(body) + "\n}\n")
    return src, P.ops


def iso_columns(which=None):
    """Columns printed by tools/dump_iso.cpp (compiled from the product's field_host.h)."""
    import subprocess
    import tempfile
    src = os.path.join(HERE, "dump_iso.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "dump_iso")
        subprocess.run(["g++", "-O2", "-o", exe, src], check=True)
        out = subprocess.run([exe] + ([which] if which else []), check=True, capture_output=True, text=True).stdout
    return [int(x, 16) for x in out.split()]


def emit_linmap_block(name, o_limb, i_limb, cols):
    """acc[i] ^= bit (32 o_limb + i) of the linear map with columns `cols` applied to the 32 planes of input
    limb i_limb (columns 32 i_limb .. 32 i_limb + 31)."""
    P = Prog()
    x = [f"X{i}" for i in range(32)]
    rows = [[j for j in range(32) if (cols[32 * i_limb + j] >> (32 * o_limb + i)) & 1] for i in range(32)]
    r = apply_linmap(P, x, rows)
    tail = [f"acc[{i}] ^= {r[i]};" for i in range(32) if r[i] != "0u"]
    import re as _re
    used = set(_re.findall(r"\bX(\d+)\b", " ".join(P.lines + tail)))
    pre = [f"const uint32_t X{i} = x[{i}];" for i in range(32) if str(i) in used]
    body = pre + P.lines + tail
    src = (f"// {name}: output limb {o_limb} <- input limb {i_limb}: {P.ops['xor']} XOR\n"
           f"GF2X_HD GF2X_INLINE void {name}_{o_limb}_{i_limb}(const uint32_t* __restrict__ x, "
           f"uint32_t* __restrict__ acc) {{\n  " + "\n  ".join(body) + "\n}\n")
    return src, P.ops["xor"]


def ipsi_columns():
    """Columns of changeRepr^-1 (tower v_k -> polynomial basis), from the product's field_host.h
    (compiled and run via tools/dump_iso.cpp), so both ipsi paths share one isomorphism."""
    import subprocess
    import tempfile
    src = os.path.join(HERE, "dump_iso.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "dump_iso")
        subprocess.run(["g++", "-O2", "-o", exe, src], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()
    cols = [int(x, 16) for x in out]
    assert len(cols) == 128
    return cols


def emit_ipsi_block(o_limb, i_limb, cols):
    """acc[i] ^= bit (32 o_limb + i) of changeRepr^-1 applied to the 32 planes of input limb i_limb."""
    P = Prog()
    x = [f"X{i}" for i in range(32)]
    rows = [[j for j in range(32) if (cols[32 * i_limb + j] >> (32 * o_limb + i)) & 1] for i in range(32)]
    r = apply_linmap(P, x, rows)
    tail = [f"acc[{i}] ^= {r[i]};" for i in range(32) if r[i] != "0u"]
    import re as _re
    used = set(_re.findall(r"\bX(\d+)\b", " ".join(P.lines + tail)))
    pre = [f"const uint32_t X{i} = x[{i}];" for i in range(32) if str(i) in used]
    body = pre + P.lines + tail
    name = f"bs_ipsi_{o_limb}_{i_limb}"
    src = (f"// changeRepr^-1 block: output limb {o_limb} <- input limb {i_limb}: {P.ops['xor']} XOR\n"
           f"GF2X_HD GF2X_INLINE void {name}(const uint32_t* __restrict__ x, uint32_t* __restrict__ acc) {{\n  "
           + "\n  ".join(body) + "\n}\n")
    return src, P.ops["xor"]


def main():
    parts = ["// GENERATED by tools/gen_bitslice.py -- do not edit.\n#pragma once\n#include <stdint.h>\n"
             "#ifndef GF2X_HD\n#define GF2X_HD\n#endif\n#ifndef GF2X_INLINE\n#define GF2X_INLINE inline\n#endif\n"]
    s, ops = emit_mul("bs_mul32", 5)
    parts.append(s)
    # products by a multiplier of a subfield (k_bottom layers whose multipliers are < 2^16 / < 2^8: Prop. 2,
    # each 16- / 8-bit block of the other factor is multiplied on its own)
    sp, opsp = emit_mul_pair("bs_mul32x2", 5)
    parts.append(sp)
    print("bs_mul32x2 ops", opsp, file=sys.stderr)
    s16, ops16 = emit_mul("bs_mul16", 4)
    parts.append(s16)
    s8, ops8 = emit_mul("bs_mul8", 3)
    parts.append(s8)
    print("bs_mul16 ops", ops16, "bs_mul8 ops", ops8, file=sys.stderr)
    v31 = 1 << 31
    s2, _ = emit_const("bs_mul_v31", v31, 5)
    parts.append(s2)
    s3, _ = emit_const("bs_mul_v31sq", tmul(v31, v31, 5), 5)
    parts.append(s3)
    cols = ipsi_columns()
    nx = 0
    for o in range(4):
        for i in range(4):
            src, n = emit_ipsi_block(o, i, cols)
            parts.append(src)
            nx += n
    # w = 128 (TGF(2^256)): changeRepr 128 -> 256 bits (4 x 8 blocks) and changeRepr^-1 256 -> 256 (8 x 8)
    c256 = iso_columns("psi256")
    assert len(c256) == 128
    n256 = 0
    for o in range(8):
        for i in range(4):
            src, n = emit_linmap_block("bs_psi256", o, i, c256)
            parts.append(src)
            n256 += n
    ci256 = iso_columns("ipsi256")
    assert len(ci256) == 256
    ni256 = 0
    for o in range(8):
        for i in range(8):
            src, n = emit_linmap_block("bs_ipsi256", o, i, ci256)
            parts.append(src)
            ni256 += n
    print("psi256 xor", n256, "ipsi256 xor", ni256, file=sys.stderr)
    with open(OUT, "w") as f:
        f.write("\n".join(parts))
    print("bs_mul32 ops", ops, "ipsi blocks xor", nx, file=sys.stderr)


if __name__ == "__main__":
    main()
