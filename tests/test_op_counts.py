"""The algorithmic ALU-op count bench.py's roofline uses for k_bottom (OPS_BS_MUL32 in gf2x.cu: ALU-pipe
instructions of one bit-sliced TGF(2^32) product) is what ptxas makes of the generated circuit: compile a
kernel that runs bs_mul32 once for sm_100a (no GPU needed) and count its LOP3 instructions.  Skipped when
nvcc / cuobjdump are not installed."""
import os
import re
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1708_09746_b200", "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

KERNEL = r'''
#include <stdint.h>
#define GF2X_HD __device__
#define GF2X_INLINE __forceinline__
#include "bitslice_gen.cuh"
#define KER(NAME, N)                                                                          \
__global__ void k_##NAME(const uint32_t* a, const uint32_t* b, uint32_t* r) {                  \
    uint32_t x[N], y[N], z[N];                                                                 \
    for (int i = 0; i < N; i++) { x[i] = a[threadIdx.x * 32 + i]; y[i] = b[threadIdx.x * 32 + i]; } \
    NAME(x, y, z);                                                                             \
    for (int i = 0; i < N; i++) r[threadIdx.x * 32 + i] = z[i];                                \
}
KER(bs_mul32, 32)
KER(bs_mul16, 16)
KER(bs_mul8, 8)
'''


@pytest.mark.skipif(not (os.path.exists(NVCC) and shutil.which("cuobjdump")), reason="needs nvcc and cuobjdump")
def test_bs_mul_lop3_counts_match_roofline_constants():
    src = open(os.path.join(CSRC, "gf2x.cu")).read()
    want = {"bs_mul32": float(re.search(r"#define OPS_BS_MUL32 ([0-9.]+)", src).group(1)),
            "bs_mul16": float(re.search(r"#define OPS_BS_MUL16 ([0-9.]+)", src).group(1)) / 2,
            "bs_mul8": float(re.search(r"#define OPS_BS_MUL8 ([0-9.]+)", src).group(1)) / 4}
    with tempfile.TemporaryDirectory() as d:
        cu = os.path.join(d, "k.cu")
        open(cu, "w").write(KERNEL)
        cubin = os.path.join(d, "k.cubin")
        subprocess.run([NVCC, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-I", CSRC, "-o", cubin, cu],
                       check=True, capture_output=True)
        sass = subprocess.run(["cuobjdump", "-sass", cubin], check=True, capture_output=True, text=True).stdout
    counts, fn = {}, None
    for ln in sass.splitlines():
        m = re.search(r"Function : _Z\d+k_(bs_mul\d+)", ln)
        if m:
            fn = m.group(1)
        elif fn and re.search(r"\bLOP3\.LUT\b", ln):
            counts[fn] = counts.get(fn, 0) + 1
    assert counts == want, (counts, want)
