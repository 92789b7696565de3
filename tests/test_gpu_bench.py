"""bench.py end to end on the GPU: the JSON line carries every key of the contract, with values consistent
with each other (short runs of small configs; the numbers themselves are not checked)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=900,
                         check=True)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("args", [["--config", "c1"], ["--config", "c2", "--graph"], ["--bits", str((1 << 20) + 128)]])
def test_bench_json_contract(args):
    import paper_1708_09746_b200 as G
    steps = 4
    d = run_bench(*args, "--steps", str(steps), "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["dtype"] == "u64" and d["data"] == "synthetic" and "workload" in d["config"]
    bits, batch = d["config"]["operand_bits"], d["config"]["batch"]
    assert d["value"] == pytest.approx(2 * bits * batch / (d["ms_per_step"] * 1e-3) / 1e9, rel=2e-3, abs=1e-3)
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=2e-3, abs=1e-4)   # (both rounded in the line)
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 2 * 8 * G.nwords(bits) * batch
    assert e["d2h_bytes_per_step"] == 16 * G.nwords(bits) * batch and e["unit"] == d["unit"] and e["value"] > 0
    assert d["gpu_launches"] == G.gf2x_launch_count(bits, bits, batch) * steps
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    if "--graph" in args:
        assert d["config"]["cuda_graph"] is True and d["config"]["ms_per_step_eager"] > 0
