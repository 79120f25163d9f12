"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product path.

ctypes/numpy front-end for

* ``oracle/build/liboracle.so`` — the plain-C restatement of the reference
  LLSA path (``oracle/llsa_oracle.c``), and
* ``oracle/_ref/libllsa_ref{32,64}.so`` — the UNMODIFIED reference library
  compiled from ``/root/reference/proj/src`` by ``oracle/Makefile`` with the
  thin C wrapper ``oracle/ref_capi.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package.  Both back-ends share one numpy-level interface
(:class:`Backend`) so a test can run the same check against either.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = {32: os.path.join(HERE, "_ref", "libllsa_ref32.so"),
          64: os.path.join(HERE, "_ref", "libllsa_ref64.so")}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


class RawConfig(C.Structure):
    """Mirror of oracle_config / ref_capi RawCfg / llsa_config (same layout)."""
    _fields_ = [("n", C.c_uint64), ("d", C.c_uint32), ("block_size", C.c_uint32),
                ("top_k", C.c_uint32), ("levels", C.c_uint32),
                ("enrich_levels", C.c_uint32), ("softmax_scale", C.c_float),
                ("reweight_mode", C.c_uint32), ("safe_softmax", C.c_uint32)]


@dataclass
class Config:
    """Python-side LLSAConfig (P/include/llsa/config.hpp:19-29)."""
    n: int
    d: int
    block_size: int
    top_k: int
    levels: int
    enrich_levels: int
    softmax_scale: float = 0.0
    reweight_mode: int = 0          # 0 ScaleKV, 1 LogitBias
    safe_softmax: bool = True

    def raw(self) -> RawConfig:
        return RawConfig(self.n, self.d, self.block_size, self.top_k, self.levels,
                         self.enrich_levels, self.softmax_scale, self.reweight_mode,
                         1 if self.safe_softmax else 0)

    # derived sizes (P/include/llsa/config.hpp:50-64)
    def pow_block(self, l: int) -> int:
        return self.block_size ** l

    def level_tokens(self, l: int) -> int:
        return self.n // self.pow_block(l)

    def level_blocks(self, l: int) -> int:
        return self.n // self.pow_block(l + 1)

    @property
    def fine_blocks(self) -> int:
        return self.level_blocks(0)

    @property
    def scale(self) -> float:
        if self.softmax_scale > 0:
            return float(np.float32(self.softmax_scale))
        return float(np.float32(1.0) / np.sqrt(np.float32(self.d)))

    @property
    def effective_blocks(self) -> int:
        le, L = self.enrich_levels, self.levels
        c = self.top_k * min(le + 1, L)
        if le == L:
            c += self.level_blocks(L)
        return c

    def pyramid_rows(self) -> int:
        return sum(self.level_tokens(l) for l in range(1, self.levels + 1))

    def table_rows(self) -> list[int]:
        return [self.level_blocks(l) for l in range(self.levels)]

    def split_pyramid(self, flat: np.ndarray) -> list[np.ndarray]:
        out, off = [], 0
        for l in range(1, self.levels + 1):
            r = self.level_tokens(l)
            out.append(flat[off:off + r])
            off += r
        return out

    def split_tables(self, flat: np.ndarray) -> list[np.ndarray]:
        out, off = [], 0
        for r in self.table_rows():
            out.append(flat[off:off + r * self.top_k].reshape(r, self.top_k))
            off += r * self.top_k
        return out


@dataclass
class PipelineResult:
    """Everything one unit's path produces (layouts as llsa_oracle.h)."""
    pyr_q: np.ndarray
    pyr_k: np.ndarray
    pyr_v: np.ndarray
    tables: np.ndarray
    out: np.ndarray
    row_max: np.ndarray
    row_denom: np.ndarray
    csc_offsets: np.ndarray | None = None
    csc_flat: np.ndarray | None = None
    dq: np.ndarray | None = None
    dk: np.ndarray | None = None
    dv: np.ndarray | None = None
    plan_level: np.ndarray | None = None
    plan_block: np.ndarray | None = None
    plan_weight: np.ndarray | None = None
    checksum: int | None = None
    macs: int | None = None
    stage_ms: list[float] = field(default_factory=list)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


def _chk(code: int, lib=None) -> None:
    if code:
        msg = ""
        if lib is not None and hasattr(lib, "ref_last_error"):
            msg = lib.ref_last_error().decode(errors="replace")
        raise OracleError(code, msg)


def _csc_sizes(cfg: Config) -> tuple[int, int]:
    offs = sum(cfg.level_blocks(l) + 1 for l in range(cfg.levels))
    flat = sum(cfg.level_blocks(l) * cfg.top_k for l in range(cfg.levels))
    return offs, flat


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


# --------------------------------------------------------------------------
# The C restatement
# --------------------------------------------------------------------------
class OracleC:
    """The C restatement (``oracle/llsa_oracle.c``), single-threaded."""

    kind = "port"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        cfgp = C.POINTER(RawConfig)
        L.oracle_max_levels.argtypes = [C.c_uint64, C.c_uint32]
        L.oracle_max_levels.restype = C.c_uint32
        L.oracle_validate.argtypes = [cfgp, C.POINTER(C.c_float), C.POINTER(C.c_uint32)]
        L.oracle_gen_random.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.c_uint64, C.c_int]
        L.oracle_gen_random.restype = None
        L.oracle_build_pyramid.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.c_uint32,
                                           C.c_uint32, _f32p]
        L.oracle_pool_backward.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.c_uint32,
                                           C.c_uint32, _f32p]
        L.oracle_select_coarsest.argtypes = [_f32p, C.c_size_t, _f32p, C.c_size_t,
                                             C.c_size_t, C.c_uint32, C.c_float, _u32p]
        L.oracle_select_level.argtypes = [_f32p, C.c_size_t, _f32p, C.c_size_t, C.c_size_t,
                                          _u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_float, C.c_uint32, _u32p]
        L.oracle_hierarchical_topk.argtypes = [cfgp, _f32p, _f32p, _u32p,
                                               C.POINTER(C.c_uint64)]
        L.oracle_build_reorder.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p]
        L.oracle_transpose.argtypes = [_u32p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                       _u32p]
        L.oracle_build_plan.argtypes = [cfgp, _u32p, _u32p, _u32p, _f32p]
        L.oracle_forward.argtypes = [cfgp, _f32p, _f32p, _f32p, _f32p, _f32p, _u32p,
                                     _f32p, _f32p, _f32p]
        L.oracle_backward.argtypes = [cfgp, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p,
                                      _f32p, _f32p, _f32p, _u32p, _u32p, _u32p, _f32p,
                                      _f32p, _f32p]
        L.oracle_input_checksum.argtypes = [cfgp, _f32p, _f32p, _f32p]
        L.oracle_input_checksum.restype = C.c_uint64

    # -- config --------------------------------------------------------------
    def max_levels(self, n: int, b: int) -> int:
        return int(self.lib.oracle_max_levels(n, b))

    def validate(self, cfg: Config) -> tuple[int, float, int]:
        s, e = C.c_float(), C.c_uint32()
        code = self.lib.oracle_validate(C.byref(cfg.raw()), C.byref(s), C.byref(e))
        return code, float(s.value), int(e.value)

    def gen_random(self, rows: int, cols: int, seed: int, uniform: bool = False):
        out = np.empty((rows, cols), np.float32)
        self.lib.oracle_gen_random(out, rows, cols, seed, 1 if uniform else 0)
        return out

    # -- stages --------------------------------------------------------------
    def build_pyramid(self, x, b: int, levels: int) -> np.ndarray:
        x = _f32(x)
        rows = sum(x.shape[0] // b ** l for l in range(1, levels + 1))
        out = np.zeros((max(rows, 1), x.shape[1]), np.float32)
        _chk(self.lib.oracle_build_pyramid(x, x.shape[0], x.shape[1], b, levels, out))
        return out[:rows]

    def pool_backward(self, g, b: int, hops: int) -> np.ndarray:
        g = _f32(g)
        out = np.empty((g.shape[0] * b ** hops, g.shape[1]), np.float32)
        _chk(self.lib.oracle_pool_backward(g, g.shape[0], g.shape[1], b, hops, out))
        return out

    def select_coarsest(self, q, k, top_k: int, scale: float) -> np.ndarray:
        q, k = _f32(q), _f32(k)
        out = np.zeros((q.shape[0], max(top_k, 1)), np.uint32)
        _chk(self.lib.oracle_select_coarsest(q, q.shape[0], k, k.shape[0], q.shape[1],
                                             top_k, scale, out))
        return out

    def select_level(self, q, k, parent, parent_level: int, top_k: int, scale: float,
                     b: int) -> np.ndarray:
        q, k, parent = _f32(q), _f32(k), _u32(parent)
        out = np.zeros((q.shape[0], max(top_k, 1)), np.uint32)
        _chk(self.lib.oracle_select_level(q, q.shape[0], k, k.shape[0], q.shape[1], parent,
                                          parent_level, parent.shape[0], parent.shape[1],
                                          top_k, scale, b, out))
        return out

    def build_reorder(self, h: int, w: int, b: int) -> tuple[int, np.ndarray, np.ndarray]:
        fwd = np.zeros(max(h * w, 1), np.uint32)
        inv = np.zeros(max(h * w, 1), np.uint32)
        code = int(self.lib.oracle_build_reorder(h, w, b, fwd, inv))
        return code, fwd[:h * w], inv[:h * w]

    def transpose(self, idx, key_blocks: int) -> tuple[np.ndarray, np.ndarray]:
        idx = _u32(idx)
        offs = np.zeros(key_blocks + 1, np.uint32)
        flat = np.zeros(max(idx.size, 1), np.uint32)
        _chk(self.lib.oracle_transpose(idx, idx.shape[0], idx.shape[1], key_blocks,
                                       offs, flat))
        return offs, flat[:idx.size]

    def checksum(self, cfg: Config, q, k, v) -> int:
        return int(self.lib.oracle_input_checksum(C.byref(cfg.raw()), _f32(q), _f32(k),
                                                  _f32(v)))

    def run(self, cfg: Config, q, k, v, d_out=None) -> PipelineResult:
        """The whole per-unit path."""
        code, _, E = self.validate(cfg)
        _chk(code)
        q, k, v = _f32(q), _f32(k), _f32(v)
        raw = cfg.raw()
        pq = self.build_pyramid(q, cfg.block_size, cfg.levels)
        pk = self.build_pyramid(k, cfg.block_size, cfg.levels)
        pv = self.build_pyramid(v, cfg.block_size, cfg.levels)
        tables = np.zeros(sum(cfg.table_rows()) * cfg.top_k, np.uint32)
        macs = C.c_uint64(0)
        _chk(self.lib.oracle_hierarchical_topk(C.byref(raw), pq, pk, tables, C.byref(macs)))
        nfb = cfg.fine_blocks
        pl = np.zeros(nfb * E, np.uint32)
        pb = np.zeros(nfb * E, np.uint32)
        pw = np.zeros(nfb * E, np.float32)
        _chk(self.lib.oracle_build_plan(C.byref(raw), tables, pl, pb, pw))
        out = np.zeros((cfg.n, cfg.d), np.float32)
        rm = np.zeros(cfg.n, np.float32)
        rd = np.zeros(cfg.n, np.float32)
        _chk(self.lib.oracle_forward(C.byref(raw), q, k, v, pk, pv, tables, out, rm, rd))
        res = PipelineResult(pq, pk, pv, tables, out, rm, rd, plan_level=pl,
                             plan_block=pb, plan_weight=pw,
                             checksum=self.checksum(cfg, q, k, v))
        if d_out is not None:
            no, nf = _csc_sizes(cfg)
            offs = np.zeros(no, np.uint32)
            flat = np.zeros(max(nf, 1), np.uint32)
            oo = of = to = 0
            for l, t in enumerate(cfg.split_tables(tables)):
                o, f = self.transpose(t, cfg.level_blocks(l))
                offs[oo:oo + o.size] = o
                flat[of:of + f.size] = f
                oo += o.size
                of += f.size
            dq = np.zeros_like(out)
            dk = np.zeros_like(out)
            dv = np.zeros_like(out)
            _chk(self.lib.oracle_backward(C.byref(raw), _f32(d_out), out, rm, rd, q, k, v,
                                          pk, pv, tables, offs, flat, dq, dk, dv))
            res.csc_offsets, res.csc_flat = offs, flat[:nf]
            res.dq, res.dk, res.dv = dq, dk, dv
        return res


# --------------------------------------------------------------------------
# The reference itself (compiled from /root/reference sources)
# --------------------------------------------------------------------------
class Reference:
    """The unmodified reference library via ``oracle/ref_capi.cpp``."""

    kind = "reference"

    def __init__(self, bits: int = 32, path: str | None = None):
        path = path or REF_SO[bits]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where "
                                    "/root/reference is present")
        self.bits = bits
        L = self.lib = C.CDLL(path)
        cfgp = C.POINTER(RawConfig)
        opt_f = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_uint]
        L.ref_threads.restype = C.c_uint
        L.ref_max_levels.argtypes = [C.c_uint64, C.c_uint32]
        L.ref_max_levels.restype = C.c_uint32
        L.ref_validate.argtypes = [cfgp, C.POINTER(C.c_float), C.POINTER(C.c_uint32)]
        L.ref_gen_random.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.c_uint64, C.c_int]
        L.ref_gen_random.restype = None
        L.ref_build_pyramid.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.c_uint32,
                                        C.c_uint32, _f32p]
        L.ref_pool_backward.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.c_uint32,
                                        C.c_uint32, _f32p]
        L.ref_select_coarsest.argtypes = [_f32p, C.c_size_t, _f32p, C.c_size_t, C.c_size_t,
                                          C.c_uint32, C.c_float, _u32p,
                                          C.POINTER(C.c_uint64)]
        L.ref_select_level.argtypes = [_f32p, C.c_size_t, _f32p, C.c_size_t, C.c_size_t,
                                       _u32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_float, C.c_uint32, _u32p, C.POINTER(C.c_uint64)]
        L.ref_transpose.argtypes = [_u32p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p]
        L.ref_build_reorder.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p]
        L.ref_run_pipeline.argtypes = [cfgp, _f32p, _f32p, _f32p] + [opt_f] * 19
        L.ref_oracle_effective.argtypes = [cfgp, _f32p, _f32p, _f32p, _f32p]
        L.ref_oracle_dense.argtypes = [_f32p, _f32p, _f32p, C.c_size_t, C.c_size_t,
                                       C.c_float, _f32p]

    def _chk(self, code):
        _chk(code, self.lib)

    def set_threads(self, t: int) -> None:
        self.lib.ref_set_threads(t)

    def threads(self) -> int:
        return int(self.lib.ref_threads())

    def max_levels(self, n: int, b: int) -> int:
        return int(self.lib.ref_max_levels(n, b))

    def validate(self, cfg: Config) -> tuple[int, float, int]:
        s, e = C.c_float(), C.c_uint32()
        code = self.lib.ref_validate(C.byref(cfg.raw()), C.byref(s), C.byref(e))
        return code, float(s.value), int(e.value)

    def gen_random(self, rows: int, cols: int, seed: int, uniform: bool = False):
        out = np.empty((rows, cols), np.float32)
        self.lib.ref_gen_random(out, rows, cols, seed, 1 if uniform else 0)
        return out

    def build_pyramid(self, x, b: int, levels: int) -> np.ndarray:
        x = _f32(x)
        rows = sum(x.shape[0] // b ** l for l in range(1, levels + 1))
        out = np.zeros((max(rows, 1), x.shape[1]), np.float32)
        self._chk(self.lib.ref_build_pyramid(x, x.shape[0], x.shape[1], b, levels, out))
        return out[:rows]

    def pool_backward(self, g, b: int, hops: int) -> np.ndarray:
        g = _f32(g)
        out = np.empty((g.shape[0] * b ** hops, g.shape[1]), np.float32)
        self._chk(self.lib.ref_pool_backward(g, g.shape[0], g.shape[1], b, hops, out))
        return out

    def select_coarsest(self, q, k, top_k: int, scale: float) -> np.ndarray:
        q, k = _f32(q), _f32(k)
        out = np.zeros((q.shape[0], max(top_k, 1)), np.uint32)
        self._chk(self.lib.ref_select_coarsest(q, q.shape[0], k, k.shape[0], q.shape[1],
                                               top_k, scale, out, None))
        return out

    def select_level(self, q, k, parent, parent_level: int, top_k: int, scale: float,
                     b: int) -> np.ndarray:
        q, k, parent = _f32(q), _f32(k), _u32(parent)
        out = np.zeros((q.shape[0], max(top_k, 1)), np.uint32)
        self._chk(self.lib.ref_select_level(q, q.shape[0], k, k.shape[0], q.shape[1],
                                            parent, parent_level, parent.shape[0],
                                            parent.shape[1], top_k, scale, b, out, None))
        return out

    def build_reorder(self, h: int, w: int, b: int) -> tuple[int, np.ndarray, np.ndarray]:
        fwd = np.zeros(max(h * w, 1), np.uint32)
        inv = np.zeros(max(h * w, 1), np.uint32)
        code = int(self.lib.ref_build_reorder(h, w, b, fwd, inv))
        return code, fwd[:h * w], inv[:h * w]

    def transpose(self, idx, key_blocks: int) -> tuple[np.ndarray, np.ndarray]:
        idx = _u32(idx)
        offs = np.zeros(key_blocks + 1, np.uint32)
        flat = np.zeros(max(idx.size, 1), np.uint32)
        self._chk(self.lib.ref_transpose(idx, idx.shape[0], idx.shape[1], key_blocks,
                                         offs, flat))
        return offs, flat[:idx.size]

    def effective_attention(self, cfg: Config, q, k, v) -> np.ndarray:
        out = np.zeros((cfg.n, cfg.d), np.float32)
        self._chk(self.lib.ref_oracle_effective(C.byref(cfg.raw()), _f32(q), _f32(k),
                                                _f32(v), out))
        return out

    def dense_attention(self, q, k, v, scale: float) -> np.ndarray:
        q = _f32(q)
        out = np.zeros_like(q)
        self._chk(self.lib.ref_oracle_dense(q, _f32(k), _f32(v), q.shape[0], q.shape[1],
                                            scale, out))
        return out

    def run(self, cfg: Config, q, k, v, d_out=None, want_outputs: bool = True
            ) -> PipelineResult:
        code, _, E = self.validate(cfg)
        self._chk(code)
        q, k, v = _f32(q), _f32(k), _f32(v)
        P = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
        n, d = cfg.n, cfg.d
        pr = cfg.pyramid_rows()
        alloc = (lambda shape, dt: np.zeros(shape, dt)) if want_outputs else \
            (lambda shape, dt: None)
        pq, pk, pv = (alloc((pr, d), np.float32) for _ in range(3))
        tables = alloc(sum(cfg.table_rows()) * cfg.top_k, np.uint32)
        nfb = cfg.fine_blocks
        pl, pb = alloc(nfb * E, np.uint32), alloc(nfb * E, np.uint32)
        pw = alloc(nfb * E, np.float32)
        out = alloc((n, d), np.float32)
        rm, rd = alloc(n, np.float32), alloc(n, np.float32)
        chk = C.c_uint64(0)
        macs = C.c_uint64(0)
        st = (C.c_double * 8)()
        offs = flat = dq = dk = dv = None
        dO = None
        if d_out is not None:
            dO = _f32(d_out)
            no, nf = _csc_sizes(cfg)
            offs, flat = alloc(no, np.uint32), alloc(max(nf, 1), np.uint32)
            dq, dk, dv = (alloc((n, d), np.float32) for _ in range(3))
        self._chk(self.lib.ref_run_pipeline(
            C.byref(cfg.raw()), q, k, v, P(dO), P(pq), P(pk), P(pv), P(tables), P(pl),
            P(pb), P(pw), P(out), P(rm), P(rd), C.cast(C.byref(chk), C.c_void_p),
            P(offs), P(flat), P(dq), P(dk), P(dv), C.cast(C.byref(macs), C.c_void_p),
            C.cast(st, C.c_void_p)))
        res = PipelineResult(pq, pk, pv, tables, out, rm, rd, offs,
                             None if flat is None else flat[:_csc_sizes(cfg)[1]],
                             dq, dk, dv, pl, pb, pw, int(chk.value), int(macs.value),
                             list(st))
        return res


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (RNE) and widen back exactly."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return (r.astype(np.uint32)).view(np.float32).reshape(x.shape)


def unit_inputs(cfg: Config, unit: int, seed: int = 42, bf16: bool = True,
                backend=None, want_dout: bool = True):
    """SURVEY.md §8(d) inputs: q,k,v,dO = gen_random(n, d, s+4u+{0,1,2,3}),
    rounded to bf16 (RNE) for bf16 configs."""
    be = backend or OracleC()
    base = seed + 4 * unit
    outs = [be.gen_random(cfg.n, cfg.d, base + i) for i in range(4 if want_dout else 3)]
    if bf16:
        outs = [bf16_round(o) for o in outs]
    return outs


def rel_err(a, ref) -> dict:
    """max|Δ|/max|ref|, relative Frobenius, and the worst and 99th-percentile
    row-relative error over rows whose reference norm is at least 1e-3 of the
    largest row norm."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    diff = a - ref
    mx = float(np.abs(ref).max()) or 1.0
    fro = float(np.linalg.norm(diff) / (np.linalg.norm(ref) or 1.0))
    if ref.ndim == 2:
        rn = np.linalg.norm(ref, axis=1)
        keep = rn > 1e-3 * max(float(rn.max()), 1e-30)   # ignore ~zero reference rows
        rr = np.linalg.norm(diff, axis=1)[keep] / rn[keep]
        worst_row = float(rr.max()) if keep.any() else 0.0
        p99_row = float(np.percentile(rr, 99)) if keep.any() else 0.0
    else:
        worst_row = p99_row = float(np.abs(diff).max() / mx)
    return {"max_rel": float(np.abs(diff).max()) / mx, "fro": fro, "worst_row": worst_row,
            "p99_row": p99_row}


def lse(row_max, row_denom):
    return np.asarray(row_max, np.float64) + np.log(np.asarray(row_denom, np.float64))


__all__ = ["Config", "OracleC", "Reference", "PipelineResult", "OracleError",
           "bf16_round", "unit_inputs", "rel_err", "lse", "math"]
