"""ctypes binding of the qsb200 C ABI (include/qsb200.h).

The shared library is built in-tree (``paper_2009_01845_b200/libqsb200.so``) by
``__graft_entry__.build()`` / ``make -C paper_2009_01845_b200/csrc``.  There is no CPU
fallback: every numeric operation of the package goes through this library, and using it
without the library or without a CUDA device raises ``SimulationError`` immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CapacityError, ShapeError, SimulationError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libqsb200.so")

QSB_C64 = 0
QSB_C128 = 1
KERNEL_AUTO = -1
KERNEL_GENERAL = 0
KERNEL_DIAGONAL = 1
KERNEL_PERMUTATION = 2

_c_void_p = ctypes.c_void_p
_c_int = ctypes.c_int
_c_u64 = ctypes.c_uint64
_c_i64 = ctypes.c_int64
_c_double = ctypes.c_double
_c_size_t = ctypes.c_size_t

# name -> (restype, argtypes); the exported surface the tests check against include/qsb200.h
SIGNATURES = {
    "qsb_abi_version": (_c_int, []),
    "qsb_last_error": (ctypes.c_char_p, []),
    "qsb_init_basis": (_c_int, [_c_void_p, _c_int, _c_int, _c_u64, _c_void_p]),
    "qsb_init_uniform": (_c_int, [_c_void_p, _c_int, _c_int, _c_double, _c_double, _c_void_p]),
    "qsb_classify": (_c_int, [_c_void_p, _c_int]),
    "qsb_apply_matrix": (
        _c_int,
        [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_int, _c_void_p, _c_void_p, _c_int, _c_void_p],
    ),
    "qsb_apply_batch": (
        _c_int,
        [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
         _c_void_p],
    ),
    "qsb_scale": (_c_int, [_c_void_p, _c_u64, _c_int, _c_double, _c_double, _c_void_p]),
    "qsb_collapse": (_c_int, [_c_void_p, _c_u64, _c_int, _c_u64, _c_u64, _c_double, _c_void_p]),
    "qsb_expect_terms": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                                  _c_void_p]),
    "qsb_run_pass": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_void_p, _c_i64, _c_void_p]),
    "qsb_pass_max_tile_bits": (_c_int, [_c_int]),
    "qsb_norm2": (_c_int, [_c_void_p, _c_u64, _c_int, _c_void_p, _c_void_p]),
    "qsb_vdot": (_c_int, [_c_void_p, _c_void_p, _c_u64, _c_int, _c_void_p, _c_void_p]),
    "qsb_probabilities": (_c_int, [_c_void_p, _c_u64, _c_int, _c_void_p, _c_void_p]),
    "qsb_marginal": (_c_int, [_c_void_p, _c_int, _c_int, _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "qsb_marginal_scratch_doubles": (_c_u64, [_c_int, _c_int]),
    "qsb_marginal_amps": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "qsb_cumsum_normalized": (_c_int, [_c_void_p, _c_u64, _c_void_p, _c_void_p, _c_size_t, _c_void_p]),
    "qsb_cumsum_scratch_bytes": (_c_size_t, [_c_u64]),
    "qsb_cumsum": (_c_int, [_c_void_p, _c_u64, _c_void_p, _c_void_p, _c_size_t, _c_int, _c_void_p]),
    "qsb_sample_counts": (_c_int, [_c_void_p, _c_u64, _c_u64, _c_u64, _c_u64, _c_u64, _c_u64, _c_void_p, _c_void_p]),
    "qsb_cumsum_serial": (_c_int, [_c_void_p, _c_u64, _c_void_p, _c_void_p]),
    "qsb_sample": (_c_int, [_c_void_p, _c_u64, _c_u64, _c_u64, _c_u64, _c_u64, _c_u64, _c_void_p, _c_void_p]),
    "qsb_jit_available": (_c_int, [ctypes.c_char_p]),
    "qsb_jit_compile": (_c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _c_void_p, _c_void_p, _c_size_t]),
    "qsb_jit_compile_cubin": (_c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _c_void_p, _c_void_p,
                                       _c_size_t, _c_void_p, _c_size_t, _c_void_p]),
    "qsb_jit_load": (_c_int, [_c_void_p, ctypes.c_char_p, _c_void_p]),
    "qsb_jit_run_pass": (
        _c_int,
        [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_u64, _c_void_p, _c_i64, _c_void_p, _c_i64, _c_int,
         _c_int, _c_int, _c_void_p],
    ),
    "qsb_jit_run_pass_dev": (
        _c_int,
        [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_u64, _c_void_p, _c_i64, _c_void_p, _c_i64, _c_int,
         _c_int, _c_int, _c_void_p],
    ),
    "qsb_permute_qubits": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_void_p, _c_void_p]),
    "qsb_exchange_halves": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_void_p]),
    "qsb_pack_half": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_u64, _c_u64, _c_void_p, _c_void_p]),
    "qsb_unpack_half": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_u64, _c_u64, _c_void_p, _c_void_p]),
    "qsb_sample_exact_scratch_bytes": (_c_size_t, [_c_u64, _c_u64]),
    "qsb_sample_exact": (_c_int, [_c_void_p, _c_u64, _c_void_p, _c_void_p, _c_size_t, _c_u64, _c_u64, _c_u64, _c_u64,
                                  _c_u64, _c_void_p, _c_void_p]),
    "qsb_sample_exact_bsums": (_c_int, [_c_void_p, _c_void_p, _c_u64, _c_void_p, _c_void_p, _c_size_t, _c_u64, _c_u64,
                                        _c_u64, _c_u64, _c_u64, _c_void_p, _c_void_p]),
    "qsb_probabilities_block_sums": (_c_int, [_c_void_p, _c_u64, _c_int, _c_void_p, _c_void_p, _c_void_p]),
    "qsb_reduced_density": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_int, _c_void_p, _c_void_p,
                                     _c_void_p]),
    "qsb_pack_part": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_u64, _c_u64, _c_u64, _c_void_p,
                               _c_void_p]),
    "qsb_unpack_part": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_u64, _c_u64, _c_u64, _c_void_p,
                                 _c_void_p]),
    "qsb_exchange_parts": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_u64, _c_u64,
                                    _c_void_p]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load (once) and type the qsb200 shared library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise SimulationError(
                f"qsb200 CUDA library not found at {path}; run __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


_STATUS_TO_ERROR = {1: ValueError, 2: ShapeError, 3: CapacityError, 4: SimulationError}


def check(status: int, what: str = ""):
    """Map a qsb_status to the reference's exception types (errors.py)."""
    if status == 0:
        return
    msg = lib().qsb_last_error().decode(errors="replace")
    exc = _STATUS_TO_ERROR.get(int(status), SimulationError)
    raise exc(f"{what}: {msg}" if what else msg)


_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch

        _torch = torch
    return _torch


def require_cuda():
    """The package computes only on a CUDA device; fail loudly otherwise."""
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise SimulationError("qsb200 needs a CUDA device (B200); no CPU fallback exists")
    load_library()


def stream_ptr(stream=None) -> int:
    torch = torch_mod()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
