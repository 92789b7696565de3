"""Build the sm_100a shared library libgf2x_b200.so in-tree (nvcc; no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgf2x_b200.so")
SOURCES = [os.path.join(CSRC, "gf2x.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh", ".h"))] + [
    os.path.join(ROOT, "include", "gf2x.h"),
    os.path.join(HERE, "tools", "gen_bitslice.py"),
    os.path.join(HERE, "tools", "dump_iso.cpp"),
]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [*os.environ.get("GF2X_NVCC_EXTRA", "").split(), "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    gen = os.path.join(HERE, "tools", "gen_bitslice.py")
    out = os.path.join(CSRC, "bitslice_gen.cuh")
    gen_deps = [gen, os.path.join(HERE, "tools", "dump_iso.cpp"), os.path.join(CSRC, "field_host.h")]
    if force or not os.path.exists(out) or any(os.path.getmtime(out) < os.path.getmtime(d) for d in gen_deps):
        subprocess.run([sys.executable, gen], check=True)
    if force or stale():
        cmd = [NVCC, *FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *SOURCES, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(HERE, "build.log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed (see %s)" % log)
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(name: str, defines: list[str]) -> str:
    """Tuning aid: the library with extra -D flags as libgf2x_b200_<name>.so (A/B timing, tools/dev/ab_bench.py)."""
    build()
    path = os.path.join(HERE, f"libgf2x_b200_{name}.so")
    cmd = [NVCC, *[f"-D{d}" for d in defines], *FLAGS, "-I", os.path.join(ROOT, "include"), "-o", path, *SOURCES, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed for variant " + name)
    return path


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":   # --variant NAME DEF [DEF ...]
        print(build_variant(sys.argv[2], sys.argv[3:]))
        sys.exit(0)
    print(build(force="--force" in sys.argv, verbose=True))
