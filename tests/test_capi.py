"""CPU-side checks of the drop-in boundary: the sm_100a library loads, exports
every entry point include/momg_gpu.h declares, and fails loudly (no CPU
fallback) when there is no device."""
import ctypes
import os
import re

import pytest

from paper_2206_13164_b200 import momg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "momg_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(momg_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("momg_residual", "momg_fast_sweep", "momg_restrict_solution",
                 "momg_restrict_residual", "momg_fas_correct", "momg_total_mass",
                 "momg_mass_correction", "momg_residual_norm", "momg_solve_steady",
                 "momg_nmg_cycle", "momg_field_create", "momg_field_upload"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = momg.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {momg.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_host_constants_without_device():
    # c_bound = max_hermite_root(M+1) (tables.cpp:22-41; test_hermite.cpp:104-120)
    assert abs(momg.max_hermite_root(4) - (3 + 6 ** 0.5) ** 0.5) < 1e-13
    assert abs(momg.max_hermite_root(2) - 1.0) < 1e-14


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", "x") != "x" and False, reason="")
def test_no_device_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(momg.DeviceUnavailable):
        momg.CellField(momg.Grid2D.uniform(4, 4), 3)
