"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads and
exports every entry point declared in include/adaptchi_b200.h; without a GPU
it fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2604_03960_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "adaptchi_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|int64_t)\s+(achi_\w+)\s*\(", text, re.M)))


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ("achi_ctx_create", "achi_chain_run", "achi_heff_apply", "achi_svd",
              "achi_bond_select", "achi_env_update_left", "achi_eigs_lowest_dense"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = abi.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_struct_layouts_match_header_sizes():
    # sizes the C compiler gives the header structs (checked against ctypes mirrors)
    assert C.sizeof(abi.ModelSpec) == 48
    assert C.sizeof(abi.ControllerConfig) == 88
    assert C.sizeof(abi.DmrgConfig) == 48 + 88
    assert C.sizeof(abi.BondState) == 64
    assert C.sizeof(abi.TraceRow) == 80
    assert C.sizeof(abi.VisitRecord) == 96
    assert C.sizeof(abi.SweepRecord) == 56


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    from paper_2604_03960_b200.api import AchiError, Context
    with pytest.raises(AchiError) as ei:
        Context(0)
    assert ei.value.name == "NoDevice"
