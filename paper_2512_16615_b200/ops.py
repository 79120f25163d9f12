"""Python mirror of the reference operator API on CUDA tensors.

Each function maps 1:1 onto a reference function (P/ = /root/reference/proj)
and calls the C ABI (include/llsa_cuda.h) through ctypes; tensors are device
memory, pointers and sizes cross the boundary, nothing else.  Tensors are
unit-major: ``[units, n, d]`` (a 2-D ``[n, d]`` tensor is one unit), bf16 or
fp32 inputs, fp32 outputs (the reference's ``real``).  u32 index tables are
held in int32 tensors (all values < 2^31).

Errors are the reference's typed exceptions (``_lib.ConfigError`` …).
Argument errors raise before any work; device-detected ones
(IndexOutOfRange, NonFiniteError) raise at the ``check=True`` sync point.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check

# --------------------------------------------------------------------------
# config (P/include/llsa/config.hpp, P/src/config.cpp)
# --------------------------------------------------------------------------


@dataclass
class LLSAConfig:
    """LLSAConfig, config.hpp:19-29."""
    n: int = 0
    d: int = 0
    block_size: int = 0
    top_k: int = 0
    levels: int = 0
    enrich_levels: int = 0
    softmax_scale: float = 0.0
    reweight_mode: int = 0   # 0 ScaleKV, 1 LogitBias
    safe_softmax: bool = True

    def c(self) -> _lib.LLSAConfigC:
        return _lib.LLSAConfigC(self.n, self.d, self.block_size, self.top_k, self.levels,
                                self.enrich_levels, self.softmax_scale, self.reweight_mode,
                                1 if self.safe_softmax else 0)


@dataclass(frozen=True)
class ValidatedConfig:
    """ValidatedConfig, config.hpp:35-72 (derived accessors included)."""
    raw: LLSAConfig
    scale: float
    effective_blocks: int

    @property
    def n(self): return self.raw.n                       # noqa: E704
    @property
    def d(self): return self.raw.d                       # noqa: E704
    @property
    def block_size(self): return self.raw.block_size     # noqa: E704
    @property
    def top_k(self): return self.raw.top_k               # noqa: E704
    @property
    def levels(self): return self.raw.levels             # noqa: E704
    @property
    def enrich_levels(self): return self.raw.enrich_levels  # noqa: E704

    def pow_block(self, l: int) -> int:
        return self.block_size ** l

    def level_tokens(self, l: int) -> int:
        return self.n // self.pow_block(l)

    def level_blocks(self, l: int) -> int:
        return self.n // self.pow_block(l + 1)

    @property
    def fine_blocks(self) -> int:
        return self.level_blocks(0)

    def weight(self, l: int) -> float:
        return float(self.pow_block(l))

    @property
    def pyramid_rows(self) -> int:
        return sum(self.level_tokens(l) for l in range(1, self.levels + 1))

    @property
    def table_entries(self) -> int:
        return sum(self.level_blocks(l) * self.top_k for l in range(self.levels))

    @property
    def csc_offsets_entries(self) -> int:
        return sum(self.level_blocks(l) + 1 for l in range(self.levels))

    def c(self) -> _lib.LLSAConfigC:
        return self.raw.c()


def max_levels(n: int, block_size: int) -> int:
    """max_levels, config.cpp:54-64."""
    return int(_lib.load().llsa_max_levels(n, block_size))


def validate_config(cfg: LLSAConfig) -> ValidatedConfig:
    """validate_config, config.cpp:66-117 (raises the same typed errors)."""
    lib = _lib.load()
    s, e = C.c_float(), C.c_uint32()
    check(lib.llsa_validate_config(C.byref(cfg.c()), C.byref(s), C.byref(e)))
    return ValidatedConfig(cfg, float(s.value), int(e.value))


def effective_block_count(cfg: ValidatedConfig) -> int:
    """effective_block_count, config.cpp:119-125."""
    return cfg.effective_blocks


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.BF16
    if t.dtype == torch.float32:
        return _lib.F32
    raise _lib.ArgumentError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _as_units(x: torch.Tensor, name: str) -> torch.Tensor:
    if not x.is_cuda:
        raise _lib.ArgumentError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if x.dim() == 2:
        x = x.unsqueeze(0)
    if x.dim() != 3:
        raise _lib.ShapeMismatch(f"{name} must be [units, rows, d] or [rows, d]")
    return x.contiguous()


def _as_tables(x: torch.Tensor, cfg) -> torch.Tensor:
    """Selection tables as [units, table_entries] int32 (1-D: one unit)."""
    if not x.is_cuda:
        raise _lib.ArgumentError("tables must be a CUDA tensor (no CPU path exists)")
    x = x.reshape(1, -1) if x.dim() == 1 else x.reshape(x.shape[0], -1)
    if x.shape[1] != cfg.table_entries:
        raise _lib.ShapeMismatch(f"tables hold {x.shape[1]} entries per unit, the config "
                                 f"{cfg.table_entries}")
    return x.to(torch.int32).contiguous()


def sync_status() -> None:
    """Synchronise and raise any device-detected error (llsa_sync_status)."""
    check(_lib.load().llsa_sync_status(C.c_void_p(_stream())))


# --------------------------------------------------------------------------
# compression (P/src/pyramid.cpp)
# --------------------------------------------------------------------------


def build_pyramid(x: torch.Tensor, block_size: int, levels: int) -> torch.Tensor:
    """build_pyramid, pyramid.hpp:26-27.  Returns levels 1..L concatenated,
    fp32 ``[units, pyramid_rows, d]`` (level 0 is ``x`` itself)."""
    lib = _lib.load()
    x = _as_units(x, "x")
    units, rows, d = x.shape
    pr = int(lib.llsa_pyramid_rows(rows, block_size, levels))
    out = torch.empty((units, max(pr, 0), d), device=x.device, dtype=torch.float32)
    check(lib.llsa_build_pyramid(_ptr(x), _dtype_code(x), units, rows, d, block_size, levels,
                                 _ptr(out), _stream()))
    return out


def pyramid_levels(flat: torch.Tensor, n: int, block_size: int, levels: int) -> list:
    """Split a build_pyramid result into per-level views (levels 1..L)."""
    out, off, t = [], 0, n
    for _ in range(levels):
        t //= block_size
        out.append(flat[:, off:off + t])
        off += t
    return out


def build_reorder(height: int, width: int, block_size: int):
    """build_reorder, reorder2d.hpp:31-32: the hierarchical 2-D curve.
    Returns ``(forward, inverse)`` as uint32 numpy arrays of height*width
    entries (forward[pos] = raster index at sequence position pos)."""
    import numpy as np
    lib = _lib.load()
    size = int(height) * int(width)
    fwd = np.empty(max(size, 1), dtype=np.uint32)
    inv = np.empty(max(size, 1), dtype=np.uint32)
    check(lib.llsa_build_reorder(height, width, block_size, fwd.ctypes.data, inv.ctypes.data))
    return fwd[:size], inv[:size]


def apply_permutation(x: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
    """apply_permutation, reorder2d.hpp:38-39: ``out[..., i, :] = x[..., perm[i], :]``
    per unit, on the GPU (``perm`` = forward for raster → sequence order,
    inverse to undo it)."""
    lib = _lib.load()
    xu = _as_units(x, "x")
    units, rows, d = xu.shape
    m = perm.to(device=xu.device, dtype=torch.int32).contiguous()
    if m.numel() != rows:
        raise _lib.ShapeMismatch(f"matrix has {rows} rows, permutation covers {m.numel()}")
    out = torch.empty_like(xu)
    check(lib.llsa_apply_permutation(_ptr(xu), _dtype_code(xu), units, rows, d, _ptr(m),
                                     _ptr(out), _stream()))
    return out.view(x.shape)


def build_pyramid_permuted(x: torch.Tensor, perm: torch.Tensor, block_size: int,
                           levels: int) -> torch.Tensor:
    """``build_pyramid(apply_permutation(x, perm))`` with the gather fused into
    the level-1 pooling (no permuted copy of ``x`` is written)."""
    lib = _lib.load()
    xu = _as_units(x, "x")
    units, rows, d = xu.shape
    m = perm.to(device=xu.device, dtype=torch.int32).contiguous()
    if m.numel() != rows:
        raise _lib.ShapeMismatch(f"matrix has {rows} rows, permutation covers {m.numel()}")
    pr = int(lib.llsa_pyramid_rows(rows, block_size, levels))
    out = torch.empty((units, max(pr, 0), d), device=xu.device, dtype=torch.float32)
    check(lib.llsa_build_pyramid_permuted(_ptr(xu), _dtype_code(xu), units, rows, d, block_size,
                                          levels, _ptr(m), _ptr(out), _stream()))
    return out


def pool_backward(d_coarse: torch.Tensor, block_size: int, hops: int) -> torch.Tensor:
    """pool_backward, pyramid.hpp:31-32."""
    lib = _lib.load()
    g = _as_units(d_coarse.float(), "d_coarse")
    units, rows, d = g.shape
    out = torch.empty((units, rows * block_size ** hops, d), device=g.device,
                      dtype=torch.float32)
    check(lib.llsa_pool_backward(_ptr(g), units, rows, d, block_size, hops, _ptr(out),
                                 _stream()))
    return out


# --------------------------------------------------------------------------
# selection (P/src/selection.cpp)
# --------------------------------------------------------------------------


def select_coarsest(q_top: torch.Tensor, k_top: torch.Tensor, top_k: int,
                    scale: float) -> torch.Tensor:
    """select_coarsest, selection.hpp:47-50 → int32 ``[units, rows, K]``."""
    lib = _lib.load()
    q = _as_units(q_top.float(), "q_top")
    k = _as_units(k_top.float(), "k_top")
    if q.shape[2] != k.shape[2]:
        raise _lib.ShapeMismatch("coarsest selection: query/key widths differ")
    units, rows, d = q.shape
    out = torch.empty((units, rows, max(top_k, 1)), device=q.device, dtype=torch.int32)
    check(lib.llsa_select_coarsest(_ptr(q), _ptr(k), units, rows, k.shape[1], d, top_k, scale,
                                   _ptr(out), _stream()))
    return out


def select_level(q_level: torch.Tensor, k_level: torch.Tensor, parent: torch.Tensor,
                 parent_level: int, top_k: int, scale: float, block_size: int
                 ) -> torch.Tensor:
    """select_level, selection.hpp:57-61 → int32 ``[units, parent_rows*B, K]``."""
    lib = _lib.load()
    q = _as_units(q_level.float(), "q_level")
    k = _as_units(k_level.float(), "k_level")
    p = _as_units(parent.to(torch.int32), "parent")
    if q.shape[2] != k.shape[2]:
        raise _lib.ShapeMismatch("level selection: query/key widths differ")
    units, parent_rows, parent_k = p.shape
    if q.shape[1] != parent_rows * block_size:
        raise _lib.ShapeMismatch(f"level selection: expected {parent_rows * block_size} "
                                 f"query tokens, got {q.shape[1]}")
    out = torch.empty((units, q.shape[1], max(top_k, 1)), device=q.device, dtype=torch.int32)
    check(lib.llsa_select_level(_ptr(q), _ptr(k), _ptr(p), units, parent_level, parent_rows,
                                parent_k, k.shape[1], q.shape[2], top_k, scale, block_size,
                                _ptr(out), _stream()))
    return out


def hierarchical_topk(pyr_q: torch.Tensor, pyr_k: torch.Tensor,
                      cfg: ValidatedConfig) -> torch.Tensor:
    """hierarchical_topk, selection.hpp:64-65.  Pyramids as from
    build_pyramid; returns flat int32 tables ``[units, table_entries]``
    (per_level 0..L-1 concatenated)."""
    lib = _lib.load()
    pq = _as_units(pyr_q, "pyr_q")
    pk = _as_units(pyr_k, "pyr_k")
    if pq.shape != pk.shape or pq.shape[1] != cfg.pyramid_rows or pq.shape[2] != cfg.d:
        raise _lib.ShapeMismatch("pyramids disagree with the config")
    units = pq.shape[0]
    out = torch.empty((units, cfg.table_entries), device=pq.device, dtype=torch.int32)
    check(lib.llsa_hierarchical_topk(C.byref(cfg.c()), units, _ptr(pq), _ptr(pk), _ptr(out),
                                     _stream()))
    return out


def split_tables(tables: torch.Tensor, cfg: ValidatedConfig) -> list:
    """Flat tables → per-level ``[units, rows_l, K]`` views (per_level[l])."""
    out, off = [], 0
    for l in range(cfg.levels):
        r = cfg.level_blocks(l)
        out.append(tables[:, off:off + r * cfg.top_k].view(tables.shape[0], r, cfg.top_k))
        off += r * cfg.top_k
    return out


def dump_selection(tables: torch.Tensor, cfg: ValidatedConfig, unit: int = 0) -> str:
    """dump_selection, selection.hpp:68 / selection.cpp:181-189 format."""
    lines = []
    for l, t in enumerate(split_tables(tables, cfg)):
        rows = t[unit].cpu().tolist()
        for i, row in enumerate(rows):
            lines.append(f"level {l} / row {i}:" + "".join(f" {x}" for x in row))
    return "".join(s + "\n" for s in lines)


# --------------------------------------------------------------------------
# CSR → CSC (P/src/indexmap.cpp)
# --------------------------------------------------------------------------


def transpose_indices(idx: torch.Tensor, key_blocks: int) -> tuple:
    """transpose_indices, indexmap.hpp:32-33 → (offsets, flat) int32."""
    lib = _lib.load()
    t = _as_units(idx.to(torch.int32), "idx")
    units, rows, k = t.shape
    offs = torch.empty((units, key_blocks + 1), device=t.device, dtype=torch.int32)
    flat = torch.empty((units, max(rows * k, 1)), device=t.device, dtype=torch.int32)
    wsb = int(lib.llsa_transpose_workspace_bytes(units, rows, k, key_blocks))
    ws = torch.empty(wsb, device=t.device, dtype=torch.uint8)
    check(lib.llsa_transpose_indices(_ptr(t), units, rows, k, key_blocks, _ptr(offs),
                                     _ptr(flat), _ptr(ws), wsb, _stream()))
    return offs, flat[:, :rows * k]


def transpose_all(tables: torch.Tensor, cfg: ValidatedConfig) -> tuple:
    """transpose_all, indexmap.hpp:36-37 → flat (offsets, flat) per unit."""
    lib = _lib.load()
    t = _as_tables(tables, cfg)
    units = t.shape[0]
    no = int(lib.llsa_csc_offsets_entries(C.byref(cfg.c())))
    nf = int(lib.llsa_csc_flat_entries(C.byref(cfg.c())))
    offs = torch.empty((units, no), device=t.device, dtype=torch.int32)
    flat = torch.empty((units, nf), device=t.device, dtype=torch.int32)
    wsb = int(lib.llsa_transpose_all_workspace_bytes(C.byref(cfg.c()), units))
    ws = torch.empty(wsb, device=t.device, dtype=torch.uint8)
    check(lib.llsa_transpose_all(C.byref(cfg.c()), units, _ptr(t), _ptr(offs), _ptr(flat),
                                 _ptr(ws), wsb, _stream()))
    return offs, flat


# --------------------------------------------------------------------------
# plan, forward, backward (P/src/attention.cpp, attention_grad.cpp)
# --------------------------------------------------------------------------


def build_plan(tables: torch.Tensor, cfg: ValidatedConfig) -> tuple:
    """build_plan, attention.hpp:44-45 → (level, block, weight) each
    ``[units, fine_blocks, E]``."""
    lib = _lib.load()
    t = _as_tables(tables, cfg)
    units, E = t.shape[0], cfg.effective_blocks
    shape = (units, cfg.fine_blocks, E)
    lv = torch.empty(shape, device=t.device, dtype=torch.int32)
    bl = torch.empty(shape, device=t.device, dtype=torch.int32)
    w = torch.empty(shape, device=t.device, dtype=torch.float32)
    check(lib.llsa_build_plan(C.byref(cfg.c()), units, _ptr(t), _ptr(lv), _ptr(bl), _ptr(w),
                              _stream()))
    return lv, bl, w


@dataclass
class ForwardState:
    """ForwardState, attention.hpp:48-55 (checksum: see input_checksum)."""
    output: torch.Tensor
    row_max: torch.Tensor
    row_denom: torch.Tensor
    mul_accs: int
    input_checksum: int = 0


def _check_qkv(q, k, v, cfg):
    for name, t in (("q", q), ("k", k), ("v", v)):
        if t.shape[1] != cfg.n or t.shape[2] != cfg.d:
            raise _lib.ShapeMismatch("q/k/v must be n x d for the validated config")
    if not (q.shape == k.shape == v.shape) or not (q.dtype == k.dtype == v.dtype):
        raise _lib.ShapeMismatch("q, k, v must share shape and dtype")


def llsa_forward(q, k, v, pyr_k, pyr_v, tables, cfg: ValidatedConfig,
                 check_finite: bool = True) -> ForwardState:
    """llsa_forward, attention.hpp:65-73.  ``tables`` replaces the
    materialised plan (the kernels read the selection directly)."""
    lib = _lib.load()
    q, k, v = (_as_units(t, n) for t, n in ((q, "q"), (k, "k"), (v, "v")))
    _check_qkv(q, k, v, cfg)
    units = q.shape[0]
    pk, pv, tb = _as_units(pyr_k, "pyr_k"), _as_units(pyr_v, "pyr_v"), _as_tables(tables, cfg)
    if tb.shape[0] != units or pk.shape[0] != units or pv.shape[0] != units:
        raise _lib.ShapeMismatch("tables / pyramids must cover the same units as q, k, v")
    out = torch.empty((units, cfg.n, cfg.d), device=q.device, dtype=torch.float32)
    rm = torch.empty((units, cfg.n), device=q.device, dtype=torch.float32)
    rd = torch.empty((units, cfg.n), device=q.device, dtype=torch.float32)
    check(lib.llsa_forward(C.byref(cfg.c()), units, _dtype_code(q), _ptr(q), _ptr(k), _ptr(v),
                           _ptr(pk), _ptr(pv), _ptr(tb), _ptr(out), _ptr(rm), _ptr(rd),
                           _stream()))
    if check_finite:
        sync_status()
    return ForwardState(out, rm, rd, int(lib.llsa_forward_mul_accs(C.byref(cfg.c()))) * units)


def llsa_backward(d_out, state: ForwardState, q, k, v, pyr_k, pyr_v, tables, transposed,
                  cfg: ValidatedConfig) -> tuple:
    """llsa_backward, attention_grad.hpp:45-52 → (dq, dk, dv) fp32."""
    lib = _lib.load()
    q, k, v = (_as_units(t, n) for t, n in ((q, "q"), (k, "k"), (v, "v")))
    _check_qkv(q, k, v, cfg)
    dO = _as_units(d_out, "d_out").to(q.dtype)
    if dO.shape != q.shape:
        raise _lib.ShapeMismatch("cotangent must be n x d")
    units = q.shape[0]
    out = _as_units(state.output, "output")
    if out.shape != q.shape:
        raise _lib.ShapeMismatch("saved forward state has wrong dimensions")
    offs, flat = transposed
    dq, dk, dv = (torch.empty((units, cfg.n, cfg.d), device=q.device, dtype=torch.float32)
                  for _ in range(3))
    wsb = int(lib.llsa_backward_workspace_bytes(C.byref(cfg.c()), units))
    ws = torch.empty(wsb, device=q.device, dtype=torch.uint8)
    check(lib.llsa_backward(C.byref(cfg.c()), units, _dtype_code(q), _ptr(dO), _ptr(out),
                            _ptr(state.row_max.contiguous()), _ptr(state.row_denom.contiguous()),
                            _ptr(q), _ptr(k), _ptr(v), _ptr(_as_units(pyr_k, "pyr_k")),
                            _ptr(_as_units(pyr_v, "pyr_v")), _ptr(_as_tables(tables, cfg)),
                            _ptr(offs.contiguous()), _ptr(flat.contiguous()), _ptr(dq), _ptr(dk),
                            _ptr(dv), _ptr(ws), wsb, _stream()))
    return dq, dk, dv


def kv_backward(d_out, state: ForwardState, q, k, v, pyr_k, pyr_v, transposed,
                cfg: ValidatedConfig) -> tuple:
    """kv_backward, attention_grad.hpp:32-37 → (dk, dv) fp32."""
    lib = _lib.load()
    q, k, v = (_as_units(t, n) for t, n in ((q, "q"), (k, "k"), (v, "v")))
    _check_qkv(q, k, v, cfg)
    dO = _as_units(d_out, "d_out").to(q.dtype)
    units = q.shape[0]
    offs, flat = transposed
    dk, dv = (torch.empty((units, cfg.n, cfg.d), device=q.device, dtype=torch.float32)
              for _ in range(2))
    wsb = int(lib.llsa_backward_workspace_bytes(C.byref(cfg.c()), units))
    ws = torch.empty(wsb, device=q.device, dtype=torch.uint8)
    check(lib.llsa_kv_backward(C.byref(cfg.c()), units, _dtype_code(q), _ptr(dO),
                               _ptr(_as_units(state.output, "output")),
                               _ptr(state.row_max.contiguous()),
                               _ptr(state.row_denom.contiguous()), _ptr(q),
                               _ptr(_as_units(pyr_k, "pyr_k")), _ptr(_as_units(pyr_v, "pyr_v")),
                               _ptr(k), _ptr(v), _ptr(offs.contiguous()),
                               _ptr(flat.contiguous()), _ptr(dk), _ptr(dv), _ptr(ws), wsb,
                               _stream()))
    return dk, dv


def mask_kv_backward(d_out, state: ForwardState, q, k, v, pyr_k, pyr_v, tables,
                     cfg: ValidatedConfig) -> tuple:
    """mask_kv_backward, oracle.hpp:54-63 → (dk, dv) fp32: the kv backward with
    the key→query lookup through dense per-level block masks (the measured
    baseline of the CSC path; same result)."""
    lib = _lib.load()
    q, k, v = (_as_units(t, n) for t, n in ((q, "q"), (k, "k"), (v, "v")))
    _check_qkv(q, k, v, cfg)
    dO = _as_units(d_out, "d_out").to(q.dtype)
    units = q.shape[0]
    dk, dv = (torch.empty((units, cfg.n, cfg.d), device=q.device, dtype=torch.float32)
              for _ in range(2))
    wsb = int(lib.llsa_mask_kv_backward_workspace_bytes(C.byref(cfg.c()), units))
    ws = torch.empty(wsb, device=q.device, dtype=torch.uint8)
    check(lib.llsa_mask_kv_backward(C.byref(cfg.c()), units, _dtype_code(q), _ptr(dO),
                                    _ptr(_as_units(state.output, "output")),
                                    _ptr(state.row_max.contiguous()),
                                    _ptr(state.row_denom.contiguous()), _ptr(q),
                                    _ptr(_as_units(pyr_k, "pyr_k")),
                                    _ptr(_as_units(pyr_v, "pyr_v")), _ptr(k), _ptr(v),
                                    _ptr(_as_tables(tables, cfg)), _ptr(dk), _ptr(dv), _ptr(ws), wsb,
                                    _stream()))
    return dk, dv


# --------------------------------------------------------------------------
# fused path
# --------------------------------------------------------------------------


class LLSAHandle:
    """Owns the device scratch of one (config, units, dtype) and runs the
    whole path in two calls (llsa_handle_* in include/llsa_cuda.h)."""

    def __init__(self, cfg: LLSAConfig | ValidatedConfig, units: int,
                 dtype: torch.dtype = torch.bfloat16, device: int | None = None):
        self.lib = _lib.load()
        self.cfg = cfg if isinstance(cfg, ValidatedConfig) else validate_config(cfg)
        if dtype not in (torch.bfloat16, torch.float32):
            raise _lib.ArgumentError(f"LLSAHandle dtype must be bfloat16 or float32, got {dtype}")
        if units < 1:
            raise _lib.ArgumentError("LLSAHandle needs at least one unit")
        self.units = units
        self.dtype = dtype
        dev = torch.cuda.current_device() if device is None else device
        self.device = torch.device("cuda", dev)
        h = C.c_void_p()
        with torch.cuda.device(dev):
            check(self.lib.llsa_handle_create(C.byref(self.cfg.c()), units,
                                              _lib.BF16 if dtype == torch.bfloat16 else _lib.F32,
                                              C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self.lib.llsa_handle_destroy(h)
            self._h = None

    @property
    def uses_tensor_cores(self) -> bool:
        return bool(self.lib.llsa_handle_uses_tensor_cores(self._h))

    @property
    def last_launches(self) -> int:
        return int(self.lib.llsa_handle_last_launches(self._h))

    def enable_timing(self, on: bool = True) -> None:
        check(self.lib.llsa_handle_enable_timing(self._h, 1 if on else 0))

    def stage_times(self) -> list[tuple[str, float]]:
        """(stage, ms) of the last forward then backward (synchronises)."""
        cap = 48
        names = (C.c_char_p * cap)()
        ms = (C.c_float * cap)()
        k = int(self.lib.llsa_handle_stage_times(self._h, names, ms, cap))
        return [(names[i].decode(), float(ms[i])) for i in range(k)]

    def buffer(self, name: str) -> tuple[int, int]:
        p, b = C.c_void_p(), C.c_size_t()
        check(self.lib.llsa_handle_buffer(self._h, _lib.BUFFERS[name], C.byref(p), C.byref(b)))
        return int(p.value or 0), int(b.value)

    def view(self, name: str) -> torch.Tensor:
        """Zero-copy tensor over a handle buffer."""
        p, nbytes = self.buffer(name)
        cfg, u = self.cfg, self.units
        shapes = {"pyr_q": ((u, cfg.pyramid_rows, cfg.d), torch.float32),
                  "pyr_k": ((u, cfg.pyramid_rows, cfg.d), torch.float32),
                  "pyr_v": ((u, cfg.pyramid_rows, cfg.d), torch.float32),
                  "tables": ((u, cfg.table_entries), torch.int32),
                  "csc_offsets": ((u, cfg.csc_offsets_entries), torch.int32),
                  "csc_flat": ((u, cfg.table_entries), torch.int32),
                  "row_max": ((u, cfg.n), torch.float32),
                  "row_denom": ((u, cfg.n), torch.float32)}
        shape, dt = shapes[name]
        numel = math.prod(shape)
        storage = torch.cuda.FloatTensor if dt == torch.float32 else None  # noqa: F841
        t = _from_ptr(p, numel, dt, self.device)
        return t.view(shape)

    def _check_inputs(self, **ts) -> None:
        """Every tensor handed to the C ABI must be [units, n, d] of the
        handle's dtype on the handle's device (the C entry points take raw
        pointers and cannot check sizes themselves)."""
        shape = (self.units, self.cfg.n, self.cfg.d)
        for name, t in ts.items():
            if tuple(t.shape) != shape:
                raise _lib.ShapeMismatch(f"{name} has shape {tuple(t.shape)}, the handle "
                                         f"expects {shape}")
            if t.dtype != self.dtype:
                raise _lib.ArgumentError(f"{name} is {t.dtype}, the handle was built for "
                                         f"{self.dtype}")
            if t.device != self.device:
                raise _lib.ArgumentError(f"{name} is on {t.device}, the handle on {self.device}")

    def _check_outputs(self, dtype=torch.float32, **ts) -> None:
        shape = (self.units, self.cfg.n, self.cfg.d)
        for name, t in ts.items():
            if tuple(t.shape) != shape or t.dtype != dtype or \
                    t.device != self.device or not t.is_contiguous():
                raise _lib.ShapeMismatch(f"{name} must be a contiguous {dtype} {shape} tensor "
                                         f"on {self.device}")

    @staticmethod
    def _out_code(dtype: torch.dtype) -> int:
        if dtype == torch.float32:
            return _lib.F32
        if dtype == torch.bfloat16:
            return _lib.BF16
        raise _lib.ArgumentError(f"outputs are float32 or bfloat16, not {dtype}")

    def forward(self, q, k, v, out=None, out_dtype: torch.dtype | None = None):
        """O = attention(q, k, v): [units, n, d] in `out_dtype` (float32 default;
        bfloat16 halves the output bytes, llsa_handle_forward_ex)."""
        self._check_inputs(q=q, k=k, v=v)
        q, k, v = (t.contiguous() for t in (q, k, v))
        out_dtype = out.dtype if out is not None else (out_dtype or torch.float32)
        code = self._out_code(out_dtype)
        out = out if out is not None else torch.empty(q.shape, device=q.device, dtype=out_dtype)
        self._check_outputs(out_dtype, out=out)
        with torch.cuda.device(self.device):
            check(self.lib.llsa_handle_forward_ex(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                                  code, _stream()))
        return out

    def backward(self, d_out, q, k, v, out, dq=None, dk=None, dv=None):
        """(dq, dk, dv) in the dtype of `out` (the forward's output)."""
        self._check_inputs(d_out=d_out, q=q, k=k, v=v)
        d_out, q, k, v = (t.contiguous() for t in (d_out, q, k, v))
        odt = out.dtype
        code = self._out_code(odt)
        mk = lambda: torch.empty(q.shape, device=q.device, dtype=odt)  # noqa: E731
        dq = dq if dq is not None else mk()
        dk = dk if dk is not None else mk()
        dv = dv if dv is not None else mk()
        self._check_outputs(odt, out=out, dq=dq, dk=dk, dv=dv)
        with torch.cuda.device(self.device):
            check(self.lib.llsa_handle_backward_ex(self._h, _ptr(d_out), _ptr(q), _ptr(k),
                                                   _ptr(v), _ptr(out), _ptr(dq), _ptr(dk),
                                                   _ptr(dv), code, _stream()))
        return dq, dk, dv


def _from_ptr(ptr: int, numel: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """Non-owning tensor over device memory owned by a handle."""
    class _CAI:
        pass
    typestr = {torch.float32: "<f4", torch.int32: "<i4"}[dtype]
    o = _CAI()
    o.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr,
                                  "data": (ptr, False), "version": 3}
    return torch.as_tensor(o, device=device)
