"""The C-ABI library: it loads, exports exactly what include/densescan_b200.h
declares, fails cleanly without a GPU, and its SASS honours the no-FMA rule.

CPU-only (no kernel is executed here).
"""

from __future__ import annotations

import ctypes
import os
import re
import shutil
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "densescan_b200.h")
LIB = os.path.join(ROOT, "paper_1506_02226_b200", "libdensescan_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ds_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1506_02226_b200", "csrc")],
                       check=True)
    from paper_1506_02226_b200 import _native
    return _native.load_library()


def test_header_declares_the_binding_set():
    from paper_1506_02226_b200 import _native
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    if shutil.which("nm"):
        out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True,
                             text=True, check=True).stdout
        exported = set(re.findall(r"\sT\s(ds_\w+)", out))
        assert set(declared_symbols()) <= exported


def test_abi_version_and_build_info(lib):
    assert lib.ds_abi_version() == 1
    assert b"sm_100a" in lib.ds_build_info()


def test_context_creation_fails_cleanly_without_gpu(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    handle = ctypes.c_void_p()
    status = lib.ds_ctx_create(0, ctypes.byref(handle))
    assert status != 0 and not handle.value
    assert lib.ds_last_error()


def test_null_arguments_are_rejected(lib):
    assert lib.ds_ctx_create(0, None) == 1  # DS_EINVAL
    assert lib.ds_run_dbscan(None, None, 0, 0, 0.0, 0, 0, 0, None, None, None) == 1


def test_no_cpu_fallback_when_library_missing(tmp_path):
    from paper_1506_02226_b200 import _native
    saved = _native._lib
    _native._lib = None
    try:
        with pytest.raises(ImportError, match="no CPU fallback"):
            _native.load_library(str(tmp_path / "missing.so"))
    finally:
        _native._lib = saved


@pytest.mark.skipif(not shutil.which("cuobjdump"), reason="cuobjdump not available")
def test_sass_gate_no_fused_multiply_add_in_pair_kernels(lib):
    """Parity needs every product and sum rounded separately (SURVEY §0 finding 4):
    the eps-tile kernels contain no scalar FFMA, and every FFMA2 is an exact product
    -- its addend is the uniform register holding {-0, -0} (UnitArgs.negz, see
    mul2_exact in ds_tile.cu), never a product's consumer contracted into it (ptxas
    would be free to fuse a packed mul+add). With d >= 2 and two lane points per
    register pair (d >= 5) the products are FFMA2 with the staged coordinate broadcast,
    the sums FADD2; at d <= 4 a lane point's products are one FMUL2; the records are staged asynchronously (cp.async -> LDGSTS)."""
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    tile = [f for f in funcs if f.startswith("_ZN2ds") and "eps_unit_kernel" in f.split("\n")[0]]
    assert len(tile) >= 16
    for body in tile:
        name = body.split("\n")[0]
        assert not re.search(r"\bFFMA\b", body), name
        for ins in re.findall(r"FFMA2[^;]*;", body):
            assert re.search(r", UR\d+\.F32 ;$", ins), (name, ins)
    k2 = [f for f in tile if "eps_unit_kernelILi2ELi1EE" in f.split("\n")[0]]
    assert k2 and "FMUL2" in k2[0] and "FADD2" in k2[0]
    assert "LDGSTS" in k2[0]
    k16 = [f for f in tile if "eps_unit_kernelILi16ELi1EE" in f.split("\n")[0]]
    assert k16 and "FFMA2" in k16[0] and "FADD2" in k16[0] and "FMUL2" not in k16[0]


@pytest.mark.skipif(not shutil.which("cuobjdump"), reason="cuobjdump not available")
def test_stage3_kernels_register_budget(lib):
    """The stage-3 union kernels are latency-bound and need their occupancy: union_diag
    (512 threads) four CTAs per SM, i.e. <= 32 registers (ptxas otherwise picked 64
    and the kernel ran 40 % slower), union_links (256 threads) four, <= 64 (its
    per-group link masks need more than 48: five CTAs spilled)."""
    out = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True,
                         check=True).stdout
    regs = {}
    for name, body in re.findall(r"Function (\S+):\n\s*(REG:\d+)", out):
        regs[name] = int(body.split(":")[1])
    diag = [r for k, r in regs.items() if "union_diag_kernel" in k]
    links = [r for k, r in regs.items() if "union_links_kernel" in k]
    assert diag and max(diag) <= 32, diag
    assert links and max(links) <= 64, links
