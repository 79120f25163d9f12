"""ctypes binding of the C ABI (include/llsa_cuda.h).

This is the reference-side binding a maintainer would add:
plain pointers and sizes, no torch types.  It fails loudly when the CUDA
library is missing — there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "lib", "libllsa_cuda.so")
HEADER = os.path.join(ROOT, "include", "llsa_cuda.h")


class LLSAConfigC(C.Structure):
    """llsa_config (include/llsa_cuda.h) == LLSAConfig, config.hpp:19-29."""
    _fields_ = [("n", C.c_uint64), ("d", C.c_uint32), ("block_size", C.c_uint32),
                ("top_k", C.c_uint32), ("levels", C.c_uint32),
                ("enrich_levels", C.c_uint32), ("softmax_scale", C.c_float),
                ("reweight_mode", C.c_uint32), ("safe_softmax", C.c_uint32)]


# ---- typed errors mirroring P/include/llsa/errors.hpp -----------------------
class Error(RuntimeError):
    """llsa::Error (errors.hpp:10)."""
    code = -1


class ConfigError(Error): code = 1          # noqa: E701
class DivisibilityError(Error): code = 2    # noqa: E701
class LevelError(Error): code = 3           # noqa: E701
class TopKError(Error): code = 4            # noqa: E701
class ShapeMismatch(Error): code = 5        # noqa: E701
class IndexOutOfRange(Error): code = 6      # noqa: E701
class NonFiniteError(Error): code = 7       # noqa: E701
class StaleState(Error): code = 8           # noqa: E701
class FormatError(Error): code = 9          # noqa: E701
class IoError(Error): code = 10             # noqa: E701
class PrecisionError(Error): code = 11      # noqa: E701
class NotSquareBlock(Error): code = 12      # noqa: E701
class OracleCapExceeded(Error): code = 13   # noqa: E701
class CudaError(Error): code = 20           # noqa: E701
class Unsupported(Error): code = 21         # noqa: E701
class ArgumentError(Error): code = 22       # noqa: E701


_BY_CODE = {c.code: c for c in (ConfigError, DivisibilityError, LevelError, TopKError,
                                ShapeMismatch, IndexOutOfRange, NonFiniteError, StaleState,
                                FormatError, IoError, PrecisionError, NotSquareBlock,
                                OracleCapExceeded, CudaError, Unsupported, ArgumentError)}

F32, BF16 = 0, 1
BUFFERS = {"pyr_q": 0, "pyr_k": 1, "pyr_v": 2, "tables": 3, "csc_offsets": 4,
           "csc_flat": 5, "row_max": 6, "row_denom": 7}

_vp, _u32, _u64, _f32, _sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_float, C.c_size_t
_cfgp = C.POINTER(LLSAConfigC)

# name: (restype, argtypes) — every symbol declared in include/llsa_cuda.h
SIGNATURES = {
    "llsa_abi_version": (C.c_int, []),
    "llsa_last_error": (C.c_char_p, []),
    "llsa_status_name": (C.c_char_p, [C.c_int]),
    "llsa_sync_status": (C.c_int, [_vp]),
    "llsa_max_levels": (_u32, [_u64, _u32]),
    "llsa_validate_config": (C.c_int, [_cfgp, C.POINTER(_f32), C.POINTER(_u32)]),
    "llsa_pyramid_rows": (_u64, [_u64, _u32, _u32]),
    "llsa_table_entries": (_u64, [_cfgp]),
    "llsa_csc_offsets_entries": (_u64, [_cfgp]),
    "llsa_csc_flat_entries": (_u64, [_cfgp]),
    "llsa_select_mul_accs": (_u64, [_cfgp]),
    "llsa_forward_mul_accs": (_u64, [_cfgp]),
    "llsa_backward_mul_accs": (_u64, [_cfgp]),
    "llsa_build_pyramid": (C.c_int, [_vp, C.c_int, _u32, _u64, _u32, _u32, _u32, _vp, _vp]),
    "llsa_pool_backward": (C.c_int, [_vp, _u32, _u64, _u32, _u32, _u32, _vp, _vp]),
    "llsa_build_reorder": (C.c_int, [_u32, _u32, _u32, _vp, _vp]),
    "llsa_apply_permutation": (C.c_int, [_vp, C.c_int, _u32, _u64, _u32, _vp, _vp, _vp]),
    "llsa_build_pyramid_permuted": (C.c_int, [_vp, C.c_int, _u32, _u64, _u32, _u32, _u32, _vp,
                                              _vp, _vp]),
    "llsa_select_coarsest": (C.c_int, [_vp, _vp, _u32, _u32, _u32, _u32, _u32, _f32, _vp, _vp]),
    "llsa_select_level": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u32, _u32, _u64, _u32, _u32,
                                    _f32, _u32, _vp, _vp]),
    "llsa_hierarchical_topk": (C.c_int, [_cfgp, _u32, _vp, _vp, _vp, _vp]),
    "llsa_transpose_workspace_bytes": (_sz, [_u32, _u32, _u32, _u32]),
    "llsa_transpose_indices": (C.c_int, [_vp, _u32, _u32, _u32, _u32, _vp, _vp, _vp, _sz, _vp]),
    "llsa_transpose_all_workspace_bytes": (_sz, [_cfgp, _u32]),
    "llsa_transpose_all": (C.c_int, [_cfgp, _u32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "llsa_build_plan": (C.c_int, [_cfgp, _u32, _vp, _vp, _vp, _vp, _vp]),
    "llsa_forward": (C.c_int, [_cfgp, _u32, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                               _vp, _vp]),
    "llsa_forward_plan": (C.c_int, [_cfgp, _u32, C.c_int] + [_vp] * 8 + [_u32] + [_vp] * 4),
    "llsa_backward_plan": (C.c_int, [_cfgp, _u32, C.c_int] + [_vp] * 12 + [_u32] +
                           [_vp] * 6 + [_sz, _vp]),
    "llsa_backward_workspace_bytes": (_sz, [_cfgp, _u32]),
    "llsa_backward": (C.c_int, [_cfgp, _u32, C.c_int] + [_vp] * 16 + [_sz, _vp]),
    "llsa_kv_backward": (C.c_int, [_cfgp, _u32, C.c_int] + [_vp] * 14 + [_sz, _vp]),
    "llsa_mask_kv_backward_workspace_bytes": (_sz, [_cfgp, _u32]),
    "llsa_mask_kv_backward": (C.c_int, [_cfgp, _u32, C.c_int] + [_vp] * 13 + [_sz, _vp]),
    "llsa_handle_create": (C.c_int, [_cfgp, _u32, C.c_int, C.POINTER(_vp)]),
    "llsa_handle_destroy": (C.c_int, [_vp]),
    "llsa_handle_uses_tensor_cores": (C.c_int, [_vp]),
    "llsa_handle_forward": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "llsa_handle_backward": (C.c_int, [_vp] + [_vp] * 8 + [_vp]),
    "llsa_handle_forward_ex": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "llsa_handle_backward_ex": (C.c_int, [_vp] + [_vp] * 8 + [C.c_int, _vp]),
    "llsa_handle_buffer": (C.c_int, [_vp, C.c_int, C.POINTER(_vp), C.POINTER(_sz)]),
    "llsa_handle_last_launches": (_u32, [_vp]),
    "llsa_handle_enable_timing": (C.c_int, [_vp, C.c_int]),
    "llsa_handle_stage_times": (_u32, [_vp, C.POINTER(C.c_char_p), C.POINTER(C.c_float), _u32]),
}


def header_symbols(path: str = HEADER) -> list[str]:
    """Function names declared in include/llsa_cuda.h."""
    with open(path) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(llsa_[a-z_0-9]+)\s*\(", text)))


_LIB: C.CDLL | None = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libllsa_cuda.so and declare every entry point.  Raises if absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python __graft_entry__.py build` "
                          "(no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(code: int) -> None:
    """Raise the typed error for a non-zero llsa_status."""
    if code:
        msg = load().llsa_last_error().decode(errors="replace")
        raise _BY_CODE.get(code, Error)(msg)
