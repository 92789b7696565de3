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
__global__ void k(const uint32_t* a, const uint32_t* b, uint32_t* r) {
    uint32_t x[32], y[32], z[32];
    for (int i = 0; i < 32; i++) { x[i] = a[threadIdx.x * 32 + i]; y[i] = b[threadIdx.x * 32 + i]; }
    bs_mul32(x, y, z);
    for (int i = 0; i < 32; i++) r[threadIdx.x * 32 + i] = z[i];
}
'''


@pytest.mark.skipif(not (os.path.exists(NVCC) and shutil.which("cuobjdump")), reason="needs nvcc and cuobjdump")
def test_bs_mul32_lop3_count_matches_roofline_constant():
    src = open(os.path.join(CSRC, "gf2x.cu")).read()
    ops = float(re.search(r"#define OPS_BS_MUL32 ([0-9.]+)", src).group(1))
    with tempfile.TemporaryDirectory() as d:
        cu = os.path.join(d, "k.cu")
        open(cu, "w").write(KERNEL)
        cubin = os.path.join(d, "k.cubin")
        subprocess.run([NVCC, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-I", CSRC, "-o", cubin, cu],
                       check=True, capture_output=True)
        sass = subprocess.run(["cuobjdump", "-sass", cubin], check=True, capture_output=True, text=True).stdout
    lop3 = len(re.findall(r"\bLOP3\.LUT\b", sass))
    assert lop3 == ops, (lop3, ops)
