"""CPU-only checks of the boundary: the C-ABI library loads, exports every
function include/mpjacobi.h declares, and the ctypes structs match the header.
No compute call is made (no GPU here)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mpjacobi.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(mpj\w+|mpjacobi_\w+)\s*\(", src)
    return sorted(set(n for n in names if not n.startswith("MPJ")))


@pytest.fixture(scope="module")
def mpjlib():
    import __graft_entry__ as g
    from paper_2211_03339_b200 import build
    build.build()
    import paper_2211_03339_b200 as m
    return m


def test_header_declares_the_boundary():
    fns = declared_functions()
    for need in ("mpjacobi_eig", "mpjacobi_svd", "mpjacobi_eig_batched", "mpjacobi_jacobi_f64",
                 "mpjacobi_orth", "mpjacobi_precond", "mpjacobi_last_error"):
        assert need in fns


def test_library_exports_every_declared_symbol(mpjlib):
    L = mpjlib.lib()
    missing = [f for f in declared_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert set(mpjlib.EXPORTED) >= set(declared_functions())


def test_config_defaults_are_the_papers(mpjlib):
    c = mpjlib.default_config("eig")
    assert (c.eps_factor, c.nu_factor) == (0.1, 20.0)
    s = mpjlib.default_config("svd")
    assert (s.eps_factor, s.nu_factor, s.early_stop_ratio) == (0.1, 1.0, 2e-4)


def test_struct_sizes_match_header(mpjlib):
    # mpj_report: 4 ints, 2 long long, 2 doubles, 64 doubles, 6 doubles, 3 ints, 1 long long,
    # 64 doubles, 64 long long
    assert C.sizeof(mpjlib.mpj_report) == 4 * 4 + 2 * 8 + 2 * 8 + 64 * 8 + 6 * 8 + 3 * 4 + 4 + 8 + 64 * 8 + 64 * 8
    assert C.sizeof(mpjlib.mpj_config) == 5 * 8 + 7 * 4 + 4   # (+4: struct padding to 8)


def test_workspace_query_needs_no_gpu(mpjlib):
    L = mpjlib.lib()
    ws = L.mpjacobi_eig_workspace(1024, C.byref(mpjlib.default_config("eig")))
    # at least 4 padded fp64 matrices and 2 fp32 ones
    assert ws >= (4 * 8 + 2 * 4) * 1024 * 1024
    assert L.mpjacobi_eig_workspace(0, None) == 0


def test_product_path_does_not_import_oracle():
    """The CUDA path must never route through oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2211_03339_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "mpj_oracle" not in txt and "liboracle" not in txt, f
