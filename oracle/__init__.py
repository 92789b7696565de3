"""CPU oracle for arXiv 1708.09746 -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package.  The CUDA product path (paper_1708_09746_b200/) never imports, links or executes it,
and it shares no code, header, table or constant generator with that path.

Layers:
  * brute.py          -- O1 bit-level brute force and O5 closed forms, pure Python integers;
  * oracle.c (ctypes) -- O2 carry-less multiply (schoolbook / Karatsuba / single output word),
                         O3 the paper's Alg. 5 step by step, O4 mod-p product checks.

Parity: every function is pinned by -m "not gpu" tests (tests/test_oracle_*.py) to values the paper
prints, closed forms, invariants or brute force.  Stage-level intermediates after changeRepr are
"parity unpinned" against the paper, because the paper does not fix its isomorphism (R9);
the final product is pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile oracle.c into oracle/liboracle.so with gcc (OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", _LIB + ".tmp", _SRC]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, i32, sz = ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t
        sig = {
            "or_clmul_impl": (i32, []),
            "or_clmul_force_portable": (None, [i32]),
            "or_clmul64": (None, [u64, u64, _u64p, _u64p]),
            "or_clmul64_portable": (None, [u64, u64, _u64p, _u64p]),
            "or_mul_schoolbook": (None, [_u64p, sz, _u64p, sz, _u64p]),
            "or_mul_karatsuba": (None, [_u64p, _u64p, sz, _u64p]),
            "or_mul_word": (u64, [_u64p, sz, _u64p, sz, sz]),
            "or_tower_mul": (None, [_u64p, _u64p, i32, _u64p]),
            "or_tower_mul_bits": (None, [_u64p, _u64p, i32, _u64p]),
            "or_gf256_generator": (i32, []),
            "or_s_eval": (None, [i32, _u64p, _u64p]),
            "or_gf128_mul": (None, [_u64p, _u64p, _u64p]),
            "or_psi_init": (i32, []),
            "or_psi": (None, [_u64p, _u64p]),
            "or_psi_inv": (None, [_u64p, _u64p]),
            "or_psi_generator": (None, [i32, _u64p]),
            "or_psi_columns": (None, [_u64p]),
            "or_basis_cvt": (None, [_u64p, i32, i32]),
            "or_ibasis_cvt": (None, [_u64p, i32, i32]),
            "or_cvt_trace": (i32, [i32, ctypes.POINTER(ctypes.c_long), i32]),
            "or_fft": (None, [_u64p, i32]),
            "or_ifft": (None, [_u64p, i32]),
            "or_fft_constant": (None, [i32, i32, u64, _u64p]),
            "or_fft_mult_count": (u64, [i32]),
            "or_alg5_mul": (i32, [_u64p, u64, _u64p, u64, _u64p] + [_u64p] * 7),
            "or_fft_alg4": (None, [_u64p, i32]),
            "or_alg4_mul": (i32, [_u64p, u64, _u64p, u64, _u64p, _u64p, _u64p]),
            "or_tower256_mul": (None, [_u64p, _u64p, _u64p]),
            "or_gf256p_mul": (None, [_u64p, _u64p, _u64p]),
            "or_psi256_init": (i32, []),
            "or_psi256": (None, [_u64p, _u64p]),
            "or_psi256_inv": (None, [_u64p, _u64p]),
            "or_psi256_generator": (None, [i32, _u64p]),
            "or_fft256": (None, [_u64p, i32]),
            "or_alg5_mul_w128": (i32, [_u64p, u64, _u64p, u64, _u64p] + [_u64p] * 4),
            "or_frob_eval": (i32, [_u64p, u64, i32, _u64p, i32]),
            "or_basis_cvt_bits": (None, [_u64p, i32, i32]),
            "or_frob_columns": (None, [i32, _u64p]),
            "or_frob_m": (i32, [u64, u64]),
            "or_frob_mul": (i32, [_u64p, u64, _u64p, u64, _u64p]),
            "or_is_irreducible64": (i32, [u64]),
            "or_poly_mod": (u64, [_u64p, sz, u64]),
            "or_mulmod64": (u64, [u64, u64, u64]),
            "or_num_threads": (i32, []),
            "or_set_threads": (None, [i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def _nullable(a):
    return _p(a) if a is not None else ctypes.cast(None, _u64p)


def _u128(x: int) -> np.ndarray:
    return np.array([x & 0xFFFFFFFFFFFFFFFF, (x >> 64) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)


def _int(a: np.ndarray) -> int:
    return int(a[0]) | (int(a[1]) << 64)


# ---------------------------------------------------------------- O2 carry-less multiplication
def clmul_impl() -> str:
    return "pclmulqdq" if lib().or_clmul_impl() == 1 else "shift-xor"


def clmul64(a: int, b: int, portable: bool = False) -> int:
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    f = lib().or_clmul64_portable if portable else lib().or_clmul64
    f(a, b, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value | (hi.value << 64)


def mul_schoolbook(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.zeros(len(a) + len(b), dtype=np.uint64)
    lib().or_mul_schoolbook(_p(a), len(a), _p(b), len(b), _p(c))
    return c


def mul_karatsuba(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    assert len(a) == len(b)
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.zeros(2 * len(a), dtype=np.uint64)
    lib().or_mul_karatsuba(_p(a), _p(b), len(a), _p(c))
    return c


def mul_word(a: np.ndarray, b: np.ndarray, w: int) -> int:
    """Output word w of a*b computed directly from the definition, O(n)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    return int(lib().or_mul_word(_p(a), len(a), _p(b), len(b), w))


# ---------------------------------------------------------------- O3 tower / s_k / psi
def tower_mul(a: int, b: int, level: int = 7, bits_only: bool = False) -> int:
    r = np.zeros(2, dtype=np.uint64)
    A, B = _u128(a), _u128(b)
    f = lib().or_tower_mul_bits if bits_only else lib().or_tower_mul
    f(_p(A), _p(B), level, _p(r))
    return _int(r)


def s_eval(k: int, x: int) -> int:
    r = np.zeros(2, dtype=np.uint64)
    X = _u128(x)
    lib().or_s_eval(k, _p(X), _p(r))
    return _int(r)


def gf128_mul(a: int, b: int) -> int:
    r = np.zeros(2, dtype=np.uint64)
    A, B = _u128(a), _u128(b)
    lib().or_gf128_mul(_p(A), _p(B), _p(r))
    return _int(r)


def psi(x: int) -> int:
    r = np.zeros(2, dtype=np.uint64)
    X = _u128(x)
    lib().or_psi(_p(X), _p(r))
    return _int(r)


def psi_inv(x: int) -> int:
    r = np.zeros(2, dtype=np.uint64)
    X = _u128(x)
    lib().or_psi_inv(_p(X), _p(r))
    return _int(r)


def psi_generator(k: int) -> int:
    r = np.zeros(2, dtype=np.uint64)
    lib().or_psi_generator(k, _p(r))
    return _int(r)


def psi_columns() -> np.ndarray:
    out = np.zeros(256, dtype=np.uint64)
    lib().or_psi_columns(_p(out))
    return out.reshape(128, 2)


# ---------------------------------------------------------------- O3 transforms
def basis_cvt(f: np.ndarray, w: int = 1) -> np.ndarray:
    """Alg. 3 BasisCvt on 2^m units of w words; returns a new array."""
    f = np.array(f, dtype=np.uint64, copy=True).reshape(-1)
    n = len(f) // w
    m = n.bit_length() - 1
    assert 1 << m == n
    lib().or_basis_cvt(_p(f), m, w)
    return f


def ibasis_cvt(g: np.ndarray, w: int = 1) -> np.ndarray:
    g = np.array(g, dtype=np.uint64, copy=True).reshape(-1)
    n = len(g) // w
    m = n.bit_length() - 1
    assert 1 << m == n
    lib().or_ibasis_cvt(_p(g), m, w)
    return g


def cvt_trace(m: int):
    """Taylor steps of BasisCvt on 2^m units, in execution order: list of (len, K, d, xors)."""
    buf = (ctypes.c_long * (4 * 4096))()
    n = lib().or_cvt_trace(m, buf, 4096)
    return [tuple(buf[4 * i: 4 * i + 4]) for i in range(n)]


def fft(g: np.ndarray) -> np.ndarray:
    """FFT_LCH at alpha=0 on N=2^m tower elements given as (N,2) uint64."""
    g = np.array(g, dtype=np.uint64, copy=True).reshape(-1, 2)
    m = len(g).bit_length() - 1
    assert 1 << m == len(g)
    flat = np.ascontiguousarray(g.reshape(-1))
    lib().or_fft(_p(flat), m)
    return flat.reshape(-1, 2)


def ifft(e: np.ndarray) -> np.ndarray:
    e = np.array(e, dtype=np.uint64, copy=True).reshape(-1, 2)
    m = len(e).bit_length() - 1
    flat = np.ascontiguousarray(e.reshape(-1))
    lib().or_ifft(_p(flat), m)
    return flat.reshape(-1, 2)


def fft_constant(m: int, k: int, j: int) -> int:
    r = np.zeros(2, dtype=np.uint64)
    lib().or_fft_constant(m, k, j, _p(r))
    return _int(r)


def fft_mult_count(m: int) -> int:
    return int(lib().or_fft_mult_count(m))


def alg5_mul(a: np.ndarray, a_bits: int, b: np.ndarray, b_bits: int, stages: bool = False):
    """Alg. 5 binPolyMul; returns c (na+nb words) or (c, dict of stage arrays)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    na, nb = (a_bits + 63) // 64, (b_bits + 63) // 64
    assert len(a) >= na and len(b) >= nb
    c = np.zeros(na + nb, dtype=np.uint64)
    st = {}
    if stages and a_bits and b_bits:
        L = na + nb - 1
        N = 1 << max(0, (L - 1).bit_length())
        for k in ("cvt_a", "cvt_b", "fft_a", "fft_b", "prod", "ifft", "icvt"):
            st[k] = np.zeros(2 * N, dtype=np.uint64)
    args = [st.get(k) for k in ("cvt_a", "cvt_b", "fft_a", "fft_b", "prod", "ifft", "icvt")]
    err = lib().or_alg5_mul(_p(a if len(a) else np.zeros(1, np.uint64)), a_bits,
                            _p(b if len(b) else np.zeros(1, np.uint64)), b_bits, _p(c),
                            *[_nullable(x) for x in args])
    if err != 0:
        raise RuntimeError(f"oracle alg5 internal assertion failed: {err}")
    if stages:
        return c, {k: v.reshape(-1, 2) for k, v in st.items()}
    return c


# ---------------------------------------------------------------- O3, Alg. 4 (sec 3.1)
def fft_alg4(g: np.ndarray) -> np.ndarray:
    """Alg. 4's FFT_LCH over GF(2^128) polynomial basis on N=2^m elements given as (N,2) uint64."""
    g = np.array(g, dtype=np.uint64, copy=True).reshape(-1, 2)
    m = len(g).bit_length() - 1
    assert 1 << m == len(g)
    flat = np.ascontiguousarray(g.reshape(-1))
    lib().or_fft_alg4(_p(flat), m)
    return flat.reshape(-1, 2)


def alg4_mul(a: np.ndarray, a_bits: int, b: np.ndarray, b_bits: int, stages: bool = False):
    """Alg. 4 simple binPolyMul (GF(2^128) polynomial basis, dense multipliers); c or (c, stages)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    na, nb = (a_bits + 63) // 64, (b_bits + 63) // 64
    c = np.zeros(na + nb, dtype=np.uint64)
    st = {}
    if stages and a_bits and b_bits:
        L = na + nb - 1
        N = 1 << max(0, (L - 1).bit_length())
        st = {k: np.zeros(2 * N, dtype=np.uint64) for k in ("fft_a", "prod")}
    err = lib().or_alg4_mul(_p(a if len(a) else np.zeros(1, np.uint64)), a_bits,
                            _p(b if len(b) else np.zeros(1, np.uint64)), b_bits, _p(c),
                            _nullable(st.get("fft_a")), _nullable(st.get("prod")))
    if err != 0:
        raise RuntimeError(f"oracle alg4 internal assertion failed: {err}")
    if stages:
        return c, {k: v.reshape(-1, 2) for k, v in st.items()}
    return c


# ---------------------------------------------------------------- O3, App. C (Frobenius bijection)
def basis_cvt_bits(words: np.ndarray, M: int, inverse: bool = False) -> np.ndarray:
    """Alg. 3 BasisCvt (or its inverse) on 2^M GF(2) coefficients packed in 2^(M-6) words; a new array."""
    w = np.array(words, dtype=np.uint64, copy=True).reshape(-1)
    assert M >= 6 and len(w) == 1 << (M - 6)
    lib().or_basis_cvt_bits(_p(w), M, 1 if inverse else 0)
    return w


def frob_m(a_bits: int, b_bits: int) -> int:
    """log2 of the number of evaluation points the Frobenius multiply uses (128 * 2^m >= a_bits + b_bits - 1)."""
    return lib().or_frob_m(a_bits, b_bits)


def frob_eval(a: np.ndarray, a_bits: int, m: int, stage: int = 2) -> np.ndarray:
    """E_(beta_(m+64) + V_m)(a): 2^m tower elements as (2^m, 2) words (stage 1: after the 7-layer encoding)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.zeros(2 << m, dtype=np.uint64)
    if lib().or_frob_eval(_p(a if len(a) else np.zeros(1, np.uint64)), a_bits, m, _p(out), stage) != 0:
        raise ValueError("frob_eval: bad size")
    return out.reshape(-1, 2)


def frob_columns(m: int) -> list:
    """The encoding's 128 columns (images of the unit bits j) as Python ints."""
    out = np.zeros(256, dtype=np.uint64)
    lib().or_frob_columns(m, _p(out))
    return [_int(out[2 * j:2 * j + 2]) for j in range(128)]


def frob_mul(a: np.ndarray, a_bits: int, b: np.ndarray, b_bits: int) -> np.ndarray:
    """App. C multiplication through the Frobenius bijection: c (na + nb words)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.zeros((a_bits + 63) // 64 + (b_bits + 63) // 64, dtype=np.uint64)
    err = lib().or_frob_mul(_p(a if len(a) else np.zeros(1, np.uint64)), a_bits,
                            _p(b if len(b) else np.zeros(1, np.uint64)), b_bits, _p(c if len(c) else np.zeros(1, np.uint64)))
    if err != 0:
        raise RuntimeError(f"oracle frob internal assertion failed: {err}")
    return c


# ---------------------------------------------------------------- O3, w = 128 (TGF(2^256))
def _u256(x: int) -> np.ndarray:
    return np.array([(x >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(4)], dtype=np.uint64)


def _int256(a: np.ndarray) -> int:
    return sum(int(a[i]) << (64 * i) for i in range(4))


def tower256_mul(a: int, b: int) -> int:
    r = np.zeros(4, dtype=np.uint64)
    A, B = _u256(a), _u256(b)
    lib().or_tower256_mul(_p(A), _p(B), _p(r))
    return _int256(r)


def gf256p_mul(a: int, b: int) -> int:
    """GF(2^256) = GF(2)[z]/(z^256+z^10+z^5+z^2+1), polynomial basis (R20)."""
    r = np.zeros(4, dtype=np.uint64)
    A, B = _u256(a), _u256(b)
    lib().or_gf256p_mul(_p(A), _p(B), _p(r))
    return _int256(r)


def psi256(x: int) -> int:
    r = np.zeros(4, dtype=np.uint64)
    X = _u256(x)
    lib().or_psi256(_p(X), _p(r))
    return _int256(r)


def psi256_inv(x: int) -> int:
    r = np.zeros(4, dtype=np.uint64)
    X = _u256(x)
    lib().or_psi256_inv(_p(X), _p(r))
    return _int256(r)


def psi256_generator(k: int) -> int:
    r = np.zeros(4, dtype=np.uint64)
    lib().or_psi256_generator(k, _p(r))
    return _int256(r)


def fft256(g: np.ndarray) -> np.ndarray:
    """FFT_LCH at alpha=0 on N=2^m TGF(2^256) elements given as (N,4) uint64."""
    g = np.array(g, dtype=np.uint64, copy=True).reshape(-1, 4)
    m = len(g).bit_length() - 1
    assert 1 << m == len(g)
    flat = np.ascontiguousarray(g.reshape(-1))
    lib().or_fft256(_p(flat), m)
    return flat.reshape(-1, 4)


W128_STAGES = ("cvt_a", "fft_a", "prod", "icvt")


def alg5_mul_w128(a: np.ndarray, a_bits: int, b: np.ndarray, b_bits: int, stages: bool = False):
    """Alg. 5 with 128-bit blocks over TGF(2^256); returns c (na+nb words) or (c, stage arrays (N,4))."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    na, nb = (a_bits + 63) // 64, (b_bits + 63) // 64
    assert len(a) >= na and len(b) >= nb
    c = np.zeros(na + nb, dtype=np.uint64)
    st = {}
    if stages and a_bits and b_bits:
        L = (a_bits + 127) // 128 + (b_bits + 127) // 128 - 1
        N = 1 << max(0, (L - 1).bit_length())
        for k in W128_STAGES:
            st[k] = np.zeros(4 * N, dtype=np.uint64)
    err = lib().or_alg5_mul_w128(_p(a if len(a) else np.zeros(1, np.uint64)), a_bits,
                                 _p(b if len(b) else np.zeros(1, np.uint64)), b_bits, _p(c),
                                 *[_nullable(st.get(k)) for k in W128_STAGES])
    if err != 0:
        raise RuntimeError(f"oracle alg5 (w=128) internal assertion failed: {err}")
    if stages:
        return c, {k: v.reshape(-1, 4) for k, v in st.items()}
    return c


# ---------------------------------------------------------------- O4 mod-p
def is_irreducible64(r: int) -> bool:
    return bool(lib().or_is_irreducible64(r))


def poly_mod(a: np.ndarray, r: int) -> int:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    if len(a) == 0:
        return 0
    return int(lib().or_poly_mod(_p(a), len(a), r))


def mulmod64(x: int, y: int, r: int) -> int:
    return int(lib().or_mulmod64(x, y, r))


def random_irreducibles(count: int, seed: int):
    """`count` random irreducible p = x^64 + r (r(0)=1), drawn from a SplitMix64 stream."""
    from gf2x_synth import splitmix64
    out, i = [], 0
    while len(out) < count:
        cand = splitmix64(seed, 64, start=i)
        i += 64
        for r in cand:
            r = int(r) | 1
            if is_irreducible64(r):
                out.append(r)
                if len(out) == count:
                    break
    return out


def check_mod_p(a: np.ndarray, b: np.ndarray, c: np.ndarray, primes) -> bool:
    """c == a*b (mod p) for every p = x^64 + r in primes."""
    for r in primes:
        if mulmod64(poly_mod(a, r), poly_mod(b, r), r) != poly_mod(c, r):
            return False
    return True


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_threads(n: int) -> None:
    lib().or_set_threads(n)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
