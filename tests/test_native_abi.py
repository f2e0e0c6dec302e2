"""The C-ABI library loads without a GPU and exports every entry point include/qsb200.h
declares (no compute calls here)."""

import os
import re

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "qsb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qsb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_2009_01845_b200 import _native

    lib = _native.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding types every declared symbol
    assert set(syms) <= set(_native.SIGNATURES), set(syms) - set(_native.SIGNATURES)
    assert lib.qsb_abi_version() == 5


def test_pass_tile_geometry_matches_planner():
    from paper_2009_01845_b200 import _native
    from paper_2009_01845_b200.fusion import GEOMETRY

    lib = _native.load_library()
    for dt, geo in GEOMETRY.items():
        assert lib.qsb_pass_max_tile_bits(dt) == geo.K


def test_classify_matches_host_rules():
    import numpy as np

    from paper_2009_01845_b200 import _native, gates

    lib = _native.load_library()
    code = {0: gates.KernelClass.GENERAL, 1: gates.KernelClass.DIAGONAL, 2: gates.KernelClass.PERMUTATION}
    specs = [gates.H(0), gates.X(0), gates.Y(0), gates.Z(0), gates.RZ(0, 0.3), gates.RY(0, 0.3),
             gates.CNOT(0, 1), gates.CZ(0, 1), gates.SWAP(0, 1), gates.CZPow(0, 1, 0.2),
             gates.VariationalLayer(0, 1, (0.1, 0.2, 0.3, 0.4))]
    for s in specs:
        m = np.ascontiguousarray(gates.gate_matrix(s))
        t = len(s.targets)
        assert code[lib.qsb_classify(m.ctypes.data, t)] is gates.classify_kernel(m)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2009_01845_b200")
    for dirpath, _dirs, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_pass_programs_pass_the_library_header_check():
    # without a GPU the call must get past program validation and fail only at the first
    # CUDA call (status QSB_ERR_CUDA = 4), proving planner and kernel agree on the format
    import torch

    from paper_2009_01845_b200 import _native, qft_circuit
    from paper_2009_01845_b200.fusion import PassStep, plan_circuit

    if torch.cuda.is_available():
        return
    lib = _native.load_library()
    for dt in (_native.QSB_C128, _native.QSB_C64):
        plan = plan_circuit(qft_circuit(16).queue, 16, dt)
        for s in plan.steps:
            if isinstance(s, PassStep):
                rc = lib.qsb_run_pass(None, None, 16, dt, s.words.ctypes.data, len(s.words), None)
                assert rc == 4, lib.qsb_last_error()
