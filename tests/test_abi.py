"""The drop-in boundary: libdocp_cuda.so loads on a CPU-only host and exports
every entry point include/docp_cuda.h declares (no compute calls here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "docp_cuda.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(docp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_06179_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import build
        build.build_cuda()
    return _lib


def test_header_declares_the_reference_boundary():
    names = declared()
    for fn in ("docp_linearize", "docp_assemble_schur", "docp_assemble_gamma", "docp_pcg_solve",
               "docp_recover_primal", "docp_line_search", "docp_sqp_solve", "docp_backward_vjp", "docp_il_epoch",
               "docp_kkt_residual", "docp_pcg_invocations"):
        assert fn in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_ctypes_signatures_cover_the_header(lib):
    assert set(declared()) == set(lib.SIGNATURES)
    L = lib.lib()  # loads without a GPU (statically linked cudart)
    assert L.docp_abi_version() == 1


def test_host_only_entry_points_without_gpu(lib):
    import ctypes as C
    L = lib.lib()
    p = lib.Problem(lib.AFFINE_QUADRATIC, 8, 4, 100, 1.0, 0, 0, 0, 0, 0)
    assert L.docp_theta_size(C.byref(p)) == 8 + 4 + 64 + 32 + 8 + 8
    bad = lib.Problem(lib.CARTPOLE, 3, 1, 10, 0.5, 1, 0.1, 0.5, 9.81, 0.05)
    assert L.docp_theta_size(C.byref(bad)) == -1
    st = lib.Status(lib.BREAKDOWN, 8, 3, 0)
    buf = C.create_string_buffer(128)
    L.docp_format_status(C.byref(st), buf, 128)
    assert buf.value.decode() == "pcg: p'Sp <= 0 (loss of positive definiteness) at iteration 3"


def test_product_path_fails_loudly_without_the_library(tmp_path, monkeypatch):
    from paper_2510_06179_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        _lib.lib()
