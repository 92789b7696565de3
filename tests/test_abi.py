"""C-ABI boundary checks that need no GPU: the in-tree sm_100a library builds, loads, exports every
symbol include/gf2x.h declares, and answers its host-only queries (no product is computed here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gf2x.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gf2x_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1708_09746_b200 import build
    path = build.build()
    import paper_1708_09746_b200 as G
    return G.load(path)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["gf2x_mul", "gf2x_mul_batched", "gf2x_workspace_bytes", "gf2x_mul_ws", "gf2x_status_string",
              "gf2x_last_error", "gf2x_release"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
    import paper_1708_09746_b200 as G
    assert sorted(G.EXPORTS) == declared_symbols()


def test_library_is_sm100a_only(lib):
    from paper_1708_09746_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_hot_kernels_keep_their_tma_and_cluster_instructions(lib):
    """SASS of the shipped library (profiles/round2_s4_sass_tma.md): the FFT table passes and the CVT(8) node pass
    move their tiles with TMA tensor loads / stores on mbarriers, the small-product kernel uses cluster barriers."""
    from paper_1708_09746_b200 import build
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    per, fn = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        for mn in ("UTMALDG", "UTMASTG", "SYNCS", "UCGABAR_ARV"):
            if fn and mn in line:
                per.setdefault(fn, set()).add(mn)
    fft = [k for k in per if k.startswith("_Z6k_fft2")]
    assert fft and all("UTMASTG" in per[k] for k in fft)
    assert any({"UTMALDG", "SYNCS"} <= per[k] for k in fft)
    rb = [k for k in per if k.startswith("_Z12k_cvt_rb_tma")]
    assert rb and all({"UTMALDG", "UTMASTG", "SYNCS"} <= per[k] for k in rb)
    small = [k for k in per if k.startswith("_Z7k_small")]
    assert small and all("UCGABAR_ARV" in per[k] for k in small)


def test_host_only_queries(lib):
    import paper_1708_09746_b200 as G
    assert G.version().startswith("gf2x-b200")
    assert G.gf2x_workspace_bytes(0, 100) == 0
    assert G.gf2x_workspace_bytes(1 << 16, 1 << 16) > 0
    # workspace grows with N and batch
    assert G.gf2x_workspace_bytes(1 << 20, 1 << 20) > G.gf2x_workspace_bytes(1 << 16, 1 << 16)
    assert G.gf2x_workspace_bytes(1 << 14, 1 << 14, 4096) > 100 * G.gf2x_workspace_bytes(1 << 14, 1 << 14, 1)
    assert G.gf2x_launch_count(1 << 16, 1 << 16) > 0
    assert lib.gf2x_status_string(0) == b"ok"
    assert lib.gf2x_status_string(2) == b"size too big"


def test_bad_arguments_fail_without_gpu_work(lib):
    # negative batch is rejected before any device call
    r = lib.gf2x_mul_batched(None, 64, None, 64, None, -1, None)
    assert r == 1
    assert b"negative" in lib.gf2x_last_error()
    # batch 0 is a no-op
    assert lib.gf2x_mul_batched(None, 64, None, 64, None, 0, None) == 0


def test_no_oracle_in_product_path():
    # the product package must not import, link or execute oracle/
    pkg = os.path.join(ROOT, "paper_1708_09746_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
