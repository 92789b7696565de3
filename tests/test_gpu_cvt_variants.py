"""GPU parity of the conversion-pass variants (cvt.cuh), each in a subprocess (the flags are read once per
process), against the oracle's Alg. 5 / Karatsuba on the same seeded operands:
  * default: k_cvt_top (Split fused into the top K = 16 Taylor run; generic residue classes as the
    superset-sum transform over the row bits, tests/test_cvt_top_reading.py) -- checks it actually ran;
  * GF2X_NO_CVT_TOP=1: the plain residue pass + k_prep;
  * GF2X_CVT_SLAB=1: the CVT(16) slab pass on thread-block clusters (measured slower; kept opt-in);
  * GF2X_NO_FUSED_SPLIT=1: k_cvt_top without the fused Split;
  * GF2X_NO_RB_TMA=1: the register-blocked passes with cp.async tile loads instead of TMA (k_cvt_rb_tma);
  * GF2X_NO_MCOMB=1: iBasisCvt on the 128-bit tower elements followed by changeRepr^-1 + InterleavedCombine
    (the default, R28, combines first in the novel basis and converts 64-bit words)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
from gf2x_synth import operand_pair  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r'''
import json, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1708_09746_b200 as G
from gf2x_synth import operand_pair
out = {}
for bits in map(int, sys.argv[1].split(",")):
    a, b = operand_pair(bits, seed=bits % 97)
    da = torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    db = torch.from_numpy(b.view(np.int64)).cuda().view(torch.uint64)
    G.profile_enable(True)
    c = G.gf2x_mul(da, bits, db, bits)
    torch.cuda.synchronize()
    kern = sorted({r["kernel"] for r in G.profile_report()})
    G.profile_enable(False)
    out[bits] = {"words": c.cpu().view(torch.int64).numpy().view(np.uint64).tolist(), "kernels": kern}
json.dump(out, open(sys.argv[2], "w"))
'''

SIZES = [(1 << 21) + 64 * 5 - 3, 1 << 22, (1 << 23) - 64]   # m' = 15 (no K = 16 node), 16, 17 (top runs)
BIG = [1 << 24]                                               # top run with B = 3 row bits (and a slab)


def run_variant(env, sizes, tmp_path):
    out = tmp_path / "out.json"
    subprocess.run([sys.executable, "-c", _CHILD, ",".join(map(str, sizes)), str(out)], cwd=ROOT, check=True,
                   timeout=900, env={**os.environ, **env})
    return {int(k): v for k, v in json.load(open(out)).items()}


@pytest.mark.parametrize("env", [{}, {"GF2X_NO_CVT_TOP": "1"}, {"GF2X_CVT_SLAB": "1"}, {"GF2X_NO_FUSED_SPLIT": "1"},
                                 {"GF2X_NO_RB_TMA": "1"}, {"GF2X_NO_MCOMB": "1"}])
def test_cvt_variants_exact(env, tmp_path):
    res = run_variant(env, SIZES + BIG, tmp_path)
    for bits in SIZES + BIG:
        a, b = operand_pair(bits, seed=bits % 97)
        want = O.mul_karatsuba(a, b) if len(a) == len(b) and (len(a) & (len(a) - 1)) == 0 else O.alg5_mul(a, bits, b, bits)
        got = np.array(res[bits]["words"], dtype=np.uint64)
        assert np.array_equal(got, want), (env, bits)
    k = set(res[1 << 24]["kernels"])
    if not env:
        assert "k_cvt_top<u64>" in k and "k_ipsi_mcomb" in k and "k_prep" not in k
        assert not any(x.endswith("<u128>") for x in k) and "k_ipsi_bs" not in k
    if env.get("GF2X_NO_MCOMB"):
        assert "k_cvt_top<u128>" in k and "k_ipsi_bs" in k and "k_ipsi_mcomb" not in k
    if env.get("GF2X_NO_CVT_TOP"):
        assert not any(x.startswith("k_cvt_top") for x in k) and "k_prep" in k
    if env.get("GF2X_CVT_SLAB"):
        assert "k_cvt_slab<u64>" in k
    if env.get("GF2X_NO_FUSED_SPLIT"):
        assert "k_prep" in k and "k_cvt_top<u64>" in k
