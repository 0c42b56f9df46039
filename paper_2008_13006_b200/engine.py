"""TW-sparse GEMM engine on B200: the drop-in for the reference's
`tilewise.engine` hot path (engine.py:24-223), backed by libtw_b200.so.

Two levels:

* Reference-signature API (host buffers in, host buffers out):
  `gemm_tw`, `gemm_tew`, `spmm_csc`, `gemm_dense`, `flop_report`,
  `time_median` -- same arguments, return types and DimensionError
  behaviour as the reference; each call copies A to the GPU, runs the
  kernels and copies C back (COL_MAJOR DenseMatrix, i.e. the C^T buffer).
* Device API (torch CUDA tensors, no copies): `TwPlan` (a CompactTileSet
  packed and resident in HBM), `TwPlan.gemm`, `TwPlan.gemm_tew`,
  `DeviceCsc`, `spmm_csc_device`, `prep_activations`.

There is no CPU fallback: without libtw_b200.so or an sm_100 GPU every
compute call raises.  `workers` is accepted for signature compatibility
(the reference's thread count); the GPU path is one persistent launch.
"""

from __future__ import annotations

import ctypes
import os
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .matrix import CscMatrix, DenseMatrix, DimensionError, Layout, as_csc, as_dense
from .pattern import (CompactTile, CompactTileSet, _flatten_tiles, compact, dense_pattern, pack_mask_words,
                      unpack_mask_words)

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

_DT = {}
if torch is not None:
    _DT = {torch.float32: _lib.TW_F32, torch.bfloat16: _lib.TW_BF16, torch.float16: _lib.TW_F16}


_TEW_CACHE = 2  # merged TEW plans kept per base plan (one per live overlay, LRU-evicted)


def _code(dtype) -> int:
    if dtype not in _DT:
        raise ValueError(f"unsupported dtype {dtype}; use float32, bfloat16 or float16")
    return _DT[dtype]


def _stream_ptr(stream, device=None) -> int:
    """Raw stream handle; None -> the current stream of `device` (the plan's
    GPU), not of whatever device happens to be current."""
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass(frozen=True)
class FlopReport:
    """engine.py:52-58"""
    wall_time: float
    flops: int
    dense_flops: int
    ratio: float


# ------------------------------------------------------------------ plans

def _plan_args(tiles, col_range):
    k, n, g = int(tiles.k), int(tiles.n), int(tiles.g)
    c0, c1 = col_range if col_range is not None else (0, n)
    col_off, col_ids, words = _flatten_tiles(tiles.tiles, k)
    sub_off = np.zeros(len(tiles.tiles) + 1, np.int64)
    for i, t in enumerate(tiles.tiles):
        sm = t.sub_matrix
        if int(sm.layout) != int(Layout.COL_MAJOR):
            raise DimensionError("CompactTile.sub_matrix must be COL_MAJOR (pattern.py:233)")
        sub_off[i + 1] = sub_off[i] + sm.rows * sm.cols
    subs = (np.ascontiguousarray(np.concatenate([np.asarray(t.sub_matrix.data, np.float32) for t in tiles.tiles]))
            if tiles.tiles else np.zeros(1, np.float32))
    if subs.size == 0:
        subs = np.zeros(1, np.float32)
    return (k, n, g, int(c0), int(c1), col_off, col_ids, words, subs, sub_off)


# TwPlan(dense_pad=None) packs a plan dense (K4) when its live tiles keep at
# least this fraction of their rows (measured crossover).
DENSE_PAD_MIN_DENSITY = float(os.environ.get("TW_B200_DENSE_PAD_MIN", "0.55"))


def tile_density(k: int, col_off, words) -> float:
    """Kept fraction of the live tiles' rows: sum k_i n_i / (K sum n_i) over
    tiles with k_i > 0 (words = the packed row masks, one row of uint32 words
    per tile)."""
    w = np.asarray(words, dtype=np.uint32).reshape(len(col_off) - 1, -1)
    k_i = np.unpackbits(w.view(np.uint8), axis=1).sum(axis=1).astype(np.int64)
    n_i = np.diff(np.asarray(col_off, dtype=np.int64))
    live = k_i > 0
    den = int(k) * int(n_i[live].sum())
    return float((k_i * n_i)[live].sum()) / den if den else 0.0


class PackedPlan:
    """The packed image of a CompactTileSet (csrc/tw_pack.cpp): padded kept-K
    index lists, output column ids, the zero-row list (pruned columns and
    dead tiles) and the swizzled 16-bit weight image.  Host-only: built and
    inspected on any machine (tw_plan_build_host)."""

    _create = "tw_plan_build_host"
    _flags = 0  # TW_PLAN_* (device plans only: tw_plan_create_ex)

    def __init__(self, tiles: CompactTileSet, dtype: str = "bf16", col_range=None, _arrays=None):
        self._h = None
        if _arrays is not None:  # packer arrays straight from a file (formats.plan_from_files)
            k, n, g, col_off, col_ids, words, subs, sub_off = _arrays
            c0, c1 = col_range if col_range is not None else (0, n)
            n_tiles = len(col_off) - 1
        else:
            k, n, g, c0, c1, col_off, col_ids, words, subs, sub_off = _plan_args(tiles, col_range)
            n_tiles = len(tiles.tiles)
        self._tiles = tiles  # host tile set (for derived plans: gemm_tew's merged plan)
        self.k, self.n, self.g, self.col_begin, self.col_end = k, n, g, c0, c1
        self.in_code = {"bf16": _lib.TW_BF16, "fp16": _lib.TW_F16}[dtype]
        handle = ctypes.c_void_p()
        self._build(handle, k, n, g, n_tiles, col_off, col_ids, words, subs, sub_off, c0, c1)
        self._h = handle
        info = _lib.PlanInfo()
        _lib.call("tw_plan_get_info", self._h, ctypes.byref(info))
        self.info = {f: getattr(info, f) for f, _ in _lib.PlanInfo._fields_}

    @classmethod
    def _host_from_arrays(cls, k, n, g, col_off, col_ids, words, subs, sub_off, dtype="bf16", col_range=None):
        return PackedPlan(None, dtype, col_range, (int(k), int(n), int(g), col_off, col_ids, words, subs, sub_off))

    def _build(self, handle, k, n, g, nt, col_off, col_ids, words, subs, sub_off, c0, c1):
        if self._create == "tw_plan_create_ex":
            _lib.call(self._create, k, n, g, nt, _np_ptr(col_off), _np_ptr(col_ids), _np_ptr(words), _np_ptr(subs),
                      _np_ptr(sub_off), self.in_code, c0, c1, self._flags, ctypes.byref(handle))
        else:
            _lib.call(self._create, k, n, g, nt, _np_ptr(col_off), _np_ptr(col_ids), _np_ptr(words), _np_ptr(subs),
                      _np_ptr(sub_off), self.in_code, c0, c1, ctypes.byref(handle))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            try:
                _lib.lib().tw_plan_destroy(h)
            except Exception:  # interpreter teardown
                pass
            self._h = None

    @property
    def n_rows(self) -> int:
        return self.col_end - self.col_begin

    def kept_flops(self, m: int) -> int:
        return 2 * m * int(self.info["kept_elems"])

    def export(self, which: str) -> np.ndarray:
        """Host copy of a packed array: 'kidx', 'colids', 'zero_rows', 'wimg', 'tiles'."""
        sel = {"kidx": (0, np.int32), "colids": (1, np.int32), "zero_rows": (2, np.int32),
               "wimg": (3, np.uint8), "tiles": (4, np.int64)}[which]
        size = ctypes.c_int64(0)
        _lib.call("tw_plan_export", self._h, sel[0], None, ctypes.byref(size))
        out = np.zeros(max(size.value // np.dtype(sel[1]).itemsize, 1), sel[1])
        size2 = ctypes.c_int64(out.nbytes)
        _lib.call("tw_plan_export", self._h, sel[0], _np_ptr(out), ctypes.byref(size2))
        out = out[: size.value // np.dtype(sel[1]).itemsize]
        return out.reshape(-1, 8) if which == "tiles" else out


    def schedule(self, m: int, out_dtype: str = "fp32", sms: int = 148, accumulate: bool = False):
        """The static launch schedule tw_gemm uses for M tokens: per-CTA unit
        lists ((live tile, first token, 64-token quarters) rows) and zero-row
        ranges.  Zero rows are counted in pieces of <= 256 KB of one row (a
        long row is split over CTAs), so zero_off[-1] >= the number of pruned
        rows.  Host-side; returns (units[n,4], unit_off[G+1], zero_off[G+1])."""
        code = {"fp32": _lib.TW_F32, "bf16": _lib.TW_BF16, "fp16": _lib.TW_F16}[out_dtype]
        res = []
        for which in (0, 1, 2):
            size = ctypes.c_int64(0)
            _lib.call("tw_schedule_export", self._h, m, code, int(accumulate), sms, which, None, ctypes.byref(size))
            buf = np.zeros(max(size.value // 4, 1), np.int32)
            size2 = ctypes.c_int64(buf.nbytes)
            _lib.call("tw_schedule_export", self._h, m, code, int(accumulate), sms, which, _np_ptr(buf),
                      ctypes.byref(size2))
            res.append(buf[: size.value // 4])
        return res[0].reshape(-1, 4), res[1], res[2]


PRECISIONS = ("bf16", "fp32", "exact")


class TwPlan(PackedPlan):
    """A CompactTileSet packed for the persistent kernel and resident on one
    GPU (see PackedPlan for the layout).

    col_range=(c0, c1) builds a shard that computes output columns [c0, c1)
    only (rows re-based to 0) -- the unit of the N-sharded multi-GPU path.

    precision (the arithmetic the plan computes in; the reference computes in
    fp32, engine.py:152-164 / _kernels.py:13-27):
      "bf16"  -- bf16 (or fp16, `dtype`) operands on the tensor cores, fp32
                 accumulation: the north_star path (rel-L2 ~1e-7 vs the
                 reference on bf16-representable inputs, ~2e-3 on raw fp32).
      "fp32"  -- fp32-faithful on the tensor cores: operands split into bf16
                 high + low parts, A.W = Ah.Wh + Al.Wh + Ah.Wl in one TW GEMM
                 of 3 k_i rows per tile (TW_PLAN_SPLIT3); ~1e-6 relative on
                 raw fp32 data, within the reference's acceptance bar.
      "exact" -- the reference's own rounding sequence (fp32 multiply, fp32
                 add, ascending k) on CUDA cores with the fp32 weights
                 (TW_PLAN_F32_WEIGHTS): bit-identical to tilewise.gemm_tw.
    `prep(a32)` produces the matching activation operand.

    dense_pad (kernel choice, "bf16" plans of G <= 128): True packs every
    live tile with ALL K rows, the pruned ones as zero weights
    (TW_PLAN_DENSE_PAD), which runs on the CTA-pair kernel K4 (A^T by TMA
    tiles, 256 x 256 per SM pair); False keeps the kept-row gather kernel K2;
    None (default) picks K4 when the live tiles keep at least
    DENSE_PAD_MIN_DENSITY of their rows -- the near-dense regime where gathering
    the kept rows costs more than multiplying the pruned ones by zero.  Same
    products either way (a pruned weight contributes 0 * a; non-finite
    activations in a tile's pruned rows would give NaN, as in a dense GEMM)."""

    _create = "tw_plan_create_ex"

    def __init__(self, tiles: CompactTileSet, device=None, dtype=None, col_range=None, _arrays=None,
                 precision: str = "bf16", dense_pad=None):
        if torch is None:
            raise RuntimeError("torch is required for device plans")
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}, got {precision!r}")
        dtype = dtype or torch.bfloat16
        if dtype not in (torch.bfloat16, torch.float16):
            raise ValueError("plan dtype must be bfloat16 or float16")
        if precision == "fp32" and dtype != torch.bfloat16:
            raise ValueError("precision='fp32' splits operands into bf16 parts (dtype must be bfloat16)")
        self.dtype = dtype
        self.precision = precision
        self._flags = {"bf16": 0, "fp32": _lib.TW_PLAN_SPLIT3, "exact": _lib.TW_PLAN_F32_WEIGHTS}[precision]
        if dense_pad and precision != "bf16":
            raise ValueError("dense_pad applies to precision='bf16' plans")
        self._dense_pad = dense_pad if precision == "bf16" else False
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        super().__init__(tiles, "bf16" if dtype == torch.bfloat16 else "fp16", col_range, _arrays)

    @property
    def operand_dtype(self):
        """dtype of the activation operand gemm() takes."""
        return torch.float32 if self.precision == "exact" else self.dtype

    def prep(self, a32, layout=Layout.ROW_MAJOR, out=None, stream=None):
        """fp32 activations (M x K ROW_MAJOR, or the K x M buffer of a
        COL_MAJOR A) -> this plan's operand: A^T in the plan dtype ("bf16"),
        the 2K-row [hi; lo] split ("fp32"), or fp32 A^T ("exact")."""
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.precision == "bf16":
            return prep_activations(a32, layout, self.dtype, out=out, stream=stream)
        if self.precision == "exact":
            return prep_activations(a32, layout, torch.float32, out=out, stream=stream)
        return prep_activations_split(a32, layout, out=out, stream=stream)

    @classmethod
    def _from_arrays(cls, k, n, g, col_off, col_ids, words, subs, sub_off, device=None, dtype=None, col_range=None,
                     precision="bf16"):
        return cls(None, device=device, dtype=dtype, col_range=col_range, precision=precision,
                   _arrays=(int(k), int(n), int(g), col_off, col_ids, words, subs, sub_off))

    def _build(self, handle, k, n, g, nt, col_off, col_ids, words, subs, sub_off, c0, c1):
        pad = self._dense_pad
        if pad is None:
            pad = g <= 128 and tile_density(k, col_off, words) >= DENSE_PAD_MIN_DENSITY
        if pad:
            self._flags |= _lib.TW_PLAN_DENSE_PAD
        self._build_args = (k, n, g, nt, col_off, col_ids, words, subs, sub_off, c0, c1)
        with torch.cuda.device(self.device):
            super()._build(handle, k, n, g, nt, col_off, col_ids, words, subs, sub_off, c0, c1)

    @property
    def dense_padded(self) -> bool:
        """True when the plan was packed with TW_PLAN_DENSE_PAD (runs on K4)."""
        return bool(self._flags & _lib.TW_PLAN_DENSE_PAD)

    # -------------------------------------------------------------- compute
    def _check_at(self, at):
        if not (isinstance(at, torch.Tensor) and at.is_cuda):
            raise TypeError("at must be a CUDA tensor (K x M)")
        rows = int(self.info["a_rows"])
        if at.dim() != 2 or at.shape[0] != rows:
            what = "2K (the fp32 split operand, TwPlan.prep)" if self.precision == "fp32" else "K"
            raise DimensionError(f"A^T has {at.shape[0] if at.dim() == 2 else '?'} rows but the plan needs {what} = "
                                 f"{rows} (pattern K is {self.k})")
        if at.dtype != self.operand_dtype:
            raise TypeError(f"activations must be {self.operand_dtype} (plan operand dtype), got {at.dtype}")
        if at.stride(1) != 1:
            raise ValueError("A^T must be row-contiguous (M contiguous)")
        if at.device != self.device:
            raise ValueError(f"A^T is on {at.device} but the plan lives on {self.device}")
        return at.shape[1], at.stride(0)

    def _out(self, m, out, out_dtype):
        if out is None:
            return torch.empty((self.n_rows, m), dtype=out_dtype, device=self.device)
        if out.shape != (self.n_rows, m) or out.dtype != out_dtype or out.stride(1) != 1:
            raise DimensionError(f"out must be a ({self.n_rows}, {m}) row-contiguous {out_dtype} tensor")
        if out.device != self.device:
            raise ValueError(f"out is on {out.device} but the plan lives on {self.device}")
        return out

    def gemm(self, at, out=None, out_dtype=None, accumulate=False, stream=None, bias=None, relu=False,
             write_pruned=True, pdl=True):
        """C^T (N x M) = (A * expand(tiles))^T for A^T (K x M) -- engine.py:152-164.
        Pruned columns are exact zeros unless accumulate=True (then they are
        left untouched and kept columns are added into `out`).

        bias (fp32 CUDA tensor of length N) / relu: the trainer's epilogue
        (trainer.py:246-248) fused into the kernel -- relu?(C + bias) for
        every output column, pruned ones included.

        write_pruned=False (needs `out`): leave the pruned-column rows of `out`
        untouched -- for a resident output buffer whose pruned rows already
        hold their value (0, or relu?(bias)) from an earlier full call."""
        out_dtype = out_dtype or torch.float32
        if self.precision == "exact":
            if accumulate or bias is not None or relu or not write_pruned or out_dtype != torch.float32:
                raise ValueError("precision='exact' plans compute the reference's plain fp32 gemm_tw only")
            return self.gemm_exact(at, out=out, stream=stream)
        m, lda = self._check_at(at)
        if (accumulate or not write_pruned) and out is None:
            raise ValueError("accumulate=True / write_pruned=False need out")
        ct = self._out(m, out, out_dtype)
        flags = (1 if accumulate else 0) | (0 if write_pruned else 2) | (0 if pdl else 4) | (
            8 if self._dense_pad else 0)  # dense_pad=True: K4 whatever the layer size
        bias_ptr = None
        if bias is not None:
            if accumulate:
                raise ValueError("bias epilogue cannot be combined with accumulate")
            if not (isinstance(bias, torch.Tensor) and bias.is_cuda and bias.dtype == torch.float32
                    and bias.numel() == self.n and bias.is_contiguous()):
                raise DimensionError(f"bias must be a contiguous fp32 CUDA tensor of {self.n} elements")
            bias_ptr = bias.data_ptr()
        elif relu:
            raise ValueError("relu needs the bias epilogue (pass bias=zeros for a plain ReLU)")
        plan = self._for_launch(m, out_dtype)
        _lib.call("tw_gemm_ex", plan._h, at.data_ptr(), m, lda, ct.data_ptr(), ct.stride(0), _code(out_dtype),
                  flags, bias_ptr, 1 if relu else 0, _stream_ptr(stream, self.device))
        return ct

    def kernel_for(self, m: int, out_dtype=None) -> int:
        """Which kernel a gemm() of M tokens runs: 2 (K2, kept-row gathers)
        or 4 (K4, CTA pairs) -- tw_plan_kernel."""
        kern = ctypes.c_int(0)
        with torch.cuda.device(self.device):
            _lib.call("tw_plan_kernel", self._h, int(m), _code(out_dtype or torch.float32), ctypes.byref(kern))
        return kern.value

    def _for_launch(self, m: int, out_dtype):
        """An auto-padded plan (dense_pad=None) whose layer is too small to
        fill a wave of K4's CTA pairs launches its unpadded sibling on K2
        instead (built once, on first use) -- K2 on a padded plan would gather
        the pruned rows too."""
        if self._dense_pad is not None or not self.dense_padded:
            return self
        kc = self.__dict__.setdefault("_kernel_cache", {})
        key = (int(m), out_dtype)
        if key not in kc:
            kc[key] = self.kernel_for(m, out_dtype)
        if kc[key] == 4:
            return self
        alt = self.__dict__.get("_unpadded")
        if alt is None:
            k, n, g, nt, col_off, col_ids, words, subs, sub_off, c0, c1 = self._build_args
            alt = TwPlan(None, device=self.device, dtype=self.dtype, col_range=(c0, c1), precision=self.precision,
                         dense_pad=False, _arrays=(k, n, g, col_off, col_ids, words, subs, sub_off))
            self._unpadded = alt
        return alt

    def gemm_exact(self, at32, out=None, stream=None):
        """Bit-exact CUDA-core variant (fp32 activations): mm_accum's exact
        multiply/add sequence, for layout/indexing proofs."""
        if self.precision == "fp32":
            raise ValueError("gemm_exact needs a bf16 or exact plan (fp32 plans hold split rows)")
        if at32.dtype != torch.float32 or at32.shape[0] != self.k or at32.stride(1) != 1:
            raise DimensionError("gemm_exact needs fp32 A^T (K x M), row-contiguous")
        if at32.device != self.device:
            raise ValueError(f"A^T is on {at32.device} but the plan lives on {self.device}")
        m = at32.shape[1]
        ct = self._out(m, out, torch.float32)
        _lib.call("tw_gemm_exact", self._h, at32.data_ptr(), m, at32.stride(0), ct.data_ptr(), ct.stride(0),
                  _stream_ptr(stream, self.device))
        return ct

    def gemm_tew(self, at, csc: "DeviceCsc", out=None, out_dtype=None, stream=None, merged=True):
        """engine.py:184-198: TW + element-wise CSC overlay (all N columns).

        merged=True (default, the B200 path): ONE persistent TW-GEMM over a
        plan whose tiles carry the overlay too (tew_merged_tileset): each
        tile's kept-K list grows by the overlay rows of its columns and its
        weights gain the overlay values; the overlay entries of pruned
        columns form extra tiles.  The tensor cores absorb the residual, and
        there is no second pass over C^T.  merged=False: the reference's
        composition, TW-GEMM then the CSC SpMM accumulated into the same
        output (tw_gemm_tew)."""
        out_dtype = out_dtype or torch.float32
        m, lda = self._check_at(at)
        if csc.rows != self.k or csc.cols != self.n:
            raise DimensionError(f"overlay is {csc.rows}x{csc.cols}, pattern is {self.k}x{self.n}")
        if merged and csc.nnz > 0 and getattr(self, "_tiles", None) is not None and csc.host is not None:
            # merged plans keyed weakly by the overlay (dropped with it) and
            # bounded: at most _TEW_CACHE overlays keep an HBM weight image
            cache = self.__dict__.setdefault("_tew_plans", weakref.WeakKeyDictionary())
            merged_plan = cache.get(csc)
            if merged_plan is None:
                while len(cache) >= _TEW_CACHE:
                    cache.pop(next(iter(cache.keys())), None)
                ts = tew_merged_tileset(self._tiles, csc.host)
                merged_plan = TwPlan(ts, device=self.device, dtype=self.dtype, col_range=(self.col_begin, self.col_end))
                cache[csc] = merged_plan
            return merged_plan.gemm(at, out=out, out_dtype=out_dtype, stream=stream)
        ct = self._out(m, out, out_dtype)
        _lib.call("tw_gemm_tew", self._h, at.data_ptr(), m, lda, csc.col_ptr.data_ptr(), csc.row_idx.data_ptr(),
                  csc.values.data_ptr(), csc.nnz, ct.data_ptr(), ct.stride(0), _code(out_dtype),
                  _stream_ptr(stream, self.device))
        return ct


class DeviceCsc:
    """A CscMatrix (matrix.py:111-146) resident on the GPU: int32 col_ptr /
    row_idx and fp32 values (the reference's value dtype)."""

    def __init__(self, s: CscMatrix, device=None):
        s = as_csc(s)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.rows, self.cols, self.nnz = s.rows, s.cols, s.nnz
        self.host = s  # the host matrix (gemm_tew's merged plan is built from it)
        self.col_ptr = torch.from_numpy(np.asarray(s.col_ptr, np.int64).astype(np.int32)).to(dev)
        self.row_idx = torch.from_numpy(np.asarray(s.row_idx, np.int64).astype(np.int32).reshape(-1)).to(dev)
        self.values = torch.from_numpy(np.array(s.values, np.float32).reshape(-1)).to(dev)
        if self.nnz == 0:  # keep valid pointers
            self.row_idx = torch.zeros(1, dtype=torch.int32, device=dev)
            self.values = torch.zeros(1, dtype=torch.float32, device=dev)


def tew_merged_tileset(tiles: CompactTileSet, ew: CscMatrix) -> CompactTileSet:
    """The TEW layer (TW tiles + element-wise overlay, engine.py:184-198) as
    one tile set for the TW kernel.  Tile t keeps rows kept_t ∪ {overlay rows
    of its columns}, with weights expand(tiles) + S on them (TEW overlays
    restore pruned elements, pruning.py:527-561, so the sum only fills
    zeros); the overlay entries of pruned columns are grouped, ascending, into
    extra tiles of at most G columns.  C = A · (expand(tiles) + S) = tw + extra
    up to fp32 summation order."""
    ew = as_csc(ew)
    k, n, g = tiles.k, tiles.n, tiles.g
    if (ew.rows, ew.cols) != (k, n):
        raise DimensionError(f"overlay is {ew.rows}x{ew.cols}, pattern is {k}x{n}")
    dense = np.array(tiles.expand().array(), dtype=np.float32, copy=True)
    cp = np.asarray(ew.col_ptr, np.int64)
    ri = np.asarray(ew.row_idx, np.int64).reshape(-1)
    va = np.asarray(ew.values, np.float32).reshape(-1)
    col_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    np.add.at(dense, (ri, col_of), va)
    tile_of = np.full(n, -1, np.int64)
    keeps = []
    for i, t in enumerate(tiles.tiles):
        tile_of[np.asarray(t.col_ids, np.int64)] = i
        keeps.append(unpack_mask_words(t.row_mask_words, k).astype(bool))
    keeps = np.array(keeps, dtype=bool).reshape(len(tiles.tiles), k)
    sel = tile_of[col_of] >= 0
    keeps[tile_of[col_of[sel]], ri[sel]] = True
    groups = [(np.asarray(t.col_ids, np.int32), keeps[i]) for i, t in enumerate(tiles.tiles)]
    extra_cols = np.unique(col_of[~sel]).astype(np.int32)
    for j in range(0, extra_cols.size, g):
        cols = extra_cols[j: j + g]
        keep = np.zeros(k, bool)
        keep[ri[~sel][np.isin(col_of[~sel], cols)]] = True
        groups.append((cols, keep))
    out = []
    for cols, keep in groups:
        rows = np.flatnonzero(keep)
        sub = dense[np.ix_(rows, cols.astype(np.int64))]
        out.append(CompactTile(sub_matrix=DenseMatrix(rows.size, cols.size, Layout.COL_MAJOR,
                                                      np.ascontiguousarray(sub.T).reshape(-1)),
                               row_mask_words=pack_mask_words(keep), col_ids=cols))
    return CompactTileSet(k, n, g, tuple(out))


def spmm_csc_device(at, csc: DeviceCsc, out=None, out_dtype=None, accumulate=False, stream=None):
    """engine.py:167-181 on device: C^T (N x M) (+)= (A * S)^T."""
    out_dtype = out_dtype or torch.float32
    if at.dim() != 2 or at.shape[0] != csc.rows:
        raise DimensionError(f"A has {at.shape[0]} cols but S has {csc.rows} rows")
    m = at.shape[1]
    if out is None:
        out = torch.empty((csc.cols, m), dtype=out_dtype, device=at.device)
    _lib.call("tw_spmm_csc", at.data_ptr(), _code(at.dtype), csc.rows, m, at.stride(0), csc.cols,
              csc.col_ptr.data_ptr(), csc.row_idx.data_ptr(), csc.values.data_ptr(), out.data_ptr(), out.stride(0),
              _code(out.dtype), 1 if accumulate else 0, _stream_ptr(stream, at.device))
    return out


def prep_activations(a32, layout=Layout.ROW_MAJOR, dtype=None, out=None, stream=None):
    """engine.py:129 (at = A^T copy) on device with the cast fused:
    fp32 A (M x K ROW_MAJOR, or its COL_MAJOR buffer given as a K x M
    tensor) -> A^T (K x M) in `dtype`, row stride padded to a multiple of 8
    (the TMA descriptor needs 16-byte row pitch)."""
    dtype = dtype or torch.bfloat16
    if a32.dtype != torch.float32 or not a32.is_contiguous():
        raise ValueError("prep_activations takes a contiguous fp32 CUDA tensor")
    if layout == Layout.ROW_MAJOR:
        m, k = a32.shape
    else:
        k, m = a32.shape
    if out is None:
        ld = (m + 7) // 8 * 8
        out = torch.empty((k, ld), dtype=dtype, device=a32.device)[:, :m]
    _lib.call("tw_prep_activations", a32.data_ptr(), m, k, int(layout), out.data_ptr(), out.stride(0),
              _code(dtype), _stream_ptr(stream, a32.device))
    return out


def prep_activations_split(a32, layout=Layout.ROW_MAJOR, out=None, stream=None):
    """The operand of a precision='fp32' plan (TW_PLAN_SPLIT3): fp32 A ->
    [rn_bf16(A^T); rn_bf16(A^T - rn_bf16(A^T))], 2K x M bf16 (high rows then
    low rows), row stride padded to a multiple of 8."""
    if a32.dtype != torch.float32 or not a32.is_contiguous():
        raise ValueError("prep_activations_split takes a contiguous fp32 CUDA tensor")
    if layout == Layout.ROW_MAJOR:
        m, k = a32.shape
    else:
        k, m = a32.shape
    if out is None:
        ld = (m + 7) // 8 * 8
        out = torch.empty((2 * k, ld), dtype=torch.bfloat16, device=a32.device)[:, :m]
    elif out.shape != (2 * k, m) or out.dtype != torch.bfloat16 or out.stride(1) != 1:
        raise DimensionError(f"out must be a (2K, M) = ({2 * k}, {m}) row-contiguous bf16 tensor")
    _lib.call("tw_prep_activations_split", a32.data_ptr(), m, k, int(layout), out.data_ptr(), out.stride(0),
              _stream_ptr(stream, a32.device))
    return out


# ------------------------------------------------------------------ reference-signature API

# Default arithmetic of the reference-signature API.  "fp32" keeps the
# reference's fp32 contract (its acceptance bar, test_acceptance.py:63-81) on
# the tensor cores; "bf16" is the north_star fast path; "exact" reproduces
# tilewise.gemm_tw bit for bit.  INTEGRATION.md documents the choice.
DEFAULT_PRECISION = os.environ.get("TW_B200_PRECISION", "fp32")


def _precision(precision) -> str:
    p = precision or DEFAULT_PRECISION
    if p not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}, got {p!r}")
    return p


def _plan_for(tiles: CompactTileSet, device, precision: str = "bf16") -> TwPlan:
    cache = getattr(tiles, "_tw_b200_plans", None)
    if cache is None:
        cache = {}
        object.__setattr__(tiles, "_tw_b200_plans", cache)
    key = (str(device), precision)
    if key not in cache:
        cache[key] = TwPlan(tiles, device=device, precision=precision)
    return cache[key]


def _as_tileset(tiles) -> CompactTileSet:
    if isinstance(tiles, CompactTileSet):
        return tiles
    # reference CompactTileSet (duck-typed): rewrap so the plan cache can attach
    cached = getattr(tiles, "_tw_b200_wrapped", None)
    if cached is None:
        cached = CompactTileSet(int(tiles.k), int(tiles.n), int(tiles.g), tuple(tiles.tiles))
        try:
            object.__setattr__(tiles, "_tw_b200_wrapped", cached)
        except Exception:
            pass
    return cached


def _device_fp32(a: DenseMatrix, device):
    """Host DenseMatrix -> its fp32 buffer on the device (asynchronous from
    pinned memory), viewed in the buffer's own shape (M x K ROW_MAJOR, K x M
    COL_MAJOR)."""
    data = np.asarray(a.data, np.float32)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # frozen (read-only) buffers are only read here
        host = torch.from_numpy(data)
    dev = host.to(device, non_blocking=host.is_pinned())
    return dev.view(a.rows, a.cols) if a.layout == Layout.ROW_MAJOR else dev.view(a.cols, a.rows)


def _device_activations(a: DenseMatrix, device, dtype):
    """Host DenseMatrix -> device A^T (K x M) in `dtype`.  The fp32 buffer is
    copied as-is (asynchronously when it lives in pinned memory) and
    transposed / cast on the device by the prep kernel."""
    return prep_activations(_device_fp32(a, device), a.layout, dtype)


def _plan_operand(a: DenseMatrix, plan: "TwPlan", device):
    return plan.prep(_device_fp32(a, device), a.layout)


def _to_host_colmajor(ct, rows: int, cols: int, out=None) -> DenseMatrix:
    """Device C^T -> COL_MAJOR DenseMatrix.  `out` (a float32 numpy array of
    rows*cols elements, ideally in pinned memory) receives the buffer; the
    returned matrix views it."""
    if out is None:
        buf = np.empty(rows * cols, np.float32)
    else:
        buf = np.asarray(out).reshape(-1)
        if buf.dtype != np.float32 or buf.size != rows * cols:
            raise DimensionError(f"out must hold {rows * cols} float32 values")
    torch.from_numpy(buf).view(ct.shape).copy_(ct)
    return DenseMatrix(rows, cols, Layout.COL_MAJOR, buf)


def _check_workers(workers: int) -> None:
    if workers < 1:
        raise DimensionError(f"workers must be >= 1, got {workers}")  # engine.py:97-98


def gemm_tw(a: DenseMatrix, tiles: CompactTileSet, workers: int = 1, *, device=None, out=None,
            precision: str | None = None) -> DenseMatrix:
    """engine.py:152-164: C = A x expand(tiles) as a COL_MAJOR DenseMatrix.
    Pruned columns are exactly zero.  fp32 output.  `precision` (default
    DEFAULT_PRECISION, env TW_B200_PRECISION): "fp32" (split-bf16 tensor
    cores, within the reference's fp32 acceptance bar), "bf16" (bf16 operands,
    the fast path), "exact" (bit-identical to the reference) -- see TwPlan.
    `out`: optional float32 host array (M*N, pinned for full copy bandwidth)
    that receives the C^T buffer."""
    a = as_dense(a)
    tiles = _as_tileset(tiles)
    if a.cols != tiles.k:
        raise DimensionError(f"A has {a.cols} cols but pattern K is {tiles.k}")
    _check_workers(workers)
    precision = _precision(precision)
    device = device or torch.device("cuda", torch.cuda.current_device())
    if a.rows == 0:
        return DenseMatrix(0, tiles.n, Layout.COL_MAJOR, np.zeros(0, np.float32))
    plan = _plan_for(tiles, device, precision)
    if a.layout == Layout.ROW_MAJOR and a.rows >= 2 * _PIPE_CHUNK and _PIPE_ON:
        return _gemm_tw_pipelined(a, plan, device, out)
    with torch.cuda.device(device):
        ct = plan.gemm(_plan_operand(a, plan, device), out_dtype=torch.float32)
        return _to_host_colmajor(ct, a.rows, tiles.n, out)


_PIPE_CHUNK = int(os.environ.get("TW_B200_PIPE_CHUNK", "1024"))
_PIPE_ON = os.environ.get("TW_B200_PIPE", "1") != "0"
_pipe_streams: dict = {}


_pinned_staging: dict = {}


def _staging(device, shape, slot):
    """Cached pinned host staging buffers (per device / shape / slot)."""
    key = (str(device), shape, slot)
    buf = _pinned_staging.get(key)
    if buf is None:
        buf = torch.empty(shape, dtype=torch.float32, pin_memory=True)
        _pinned_staging[key] = buf
    return buf


def _gemm_tw_pipelined(a: DenseMatrix, plan: "TwPlan", device, out=None) -> DenseMatrix:
    """gemm_tw's host round trip in token chunks on three streams: the H2D
    copy + transpose/cast of chunk c+1, the TW-GEMM of chunk c and the 2-D
    D2H copy of C^T's columns for chunk c-1 overlap (PCIe is full duplex).
    Every chunk is the same kernel on a token slice (A^T columns / C^T
    columns with the full row pitch), so the result is identical to the
    one-shot path.

    Copies only overlap when they are asynchronous, i.e. between device and
    PINNED host memory.  A pageable input (or output) goes through two
    cached pinned staging buffers per direction: the host copies chunk c
    into / out of staging slot c % 2 while the GPU works on the other."""
    m, k, n = a.rows, a.cols, plan.n
    key = str(device)
    if key not in _pipe_streams:
        _pipe_streams[key] = (torch.cuda.Stream(device), torch.cuda.Stream(device))
    s_in, s_out = _pipe_streams[key]
    cur = torch.cuda.current_stream(device)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # frozen (read-only) buffers are only read here
        a_host = torch.from_numpy(np.asarray(a.data, np.float32)).view(m, k)
    if out is None:
        buf = np.empty(m * n, np.float32)
    else:
        buf = np.asarray(out).reshape(-1)
        if buf.dtype != np.float32 or buf.size != m * n:
            raise DimensionError(f"out must hold {m * n} float32 values")
    buf_t = torch.from_numpy(buf)
    pin_in, pin_out = a_host.is_pinned(), buf_t.is_pinned()
    a_dev = torch.empty((m, k), dtype=torch.float32, device=device)
    ld = (m + 7) // 8 * 8
    at = torch.empty((int(plan.info["a_rows"]), ld), dtype=plan.operand_dtype, device=device)[:, :m]
    ct = torch.empty((n, m), dtype=torch.float32, device=device)
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    ch = _PIPE_CHUNK
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]
    ev_out = [None, None]       # D2H of the chunk held in staging slot i
    pending = [None, None]      # (c0, c1) of that chunk, still to copy into buf
    buf2d = buf.reshape(n, m)

    def drain(slot):
        if pending[slot] is None:
            return
        ev_out[slot].synchronize()
        d0, d1 = pending[slot]
        buf2d[:, d0:d1] = _staging(device, (n, ch), ("out", slot)).numpy()[:, : d1 - d0]
        pending[slot] = None

    for i, c0 in enumerate(range(0, m, ch)):
        c1 = min(m, c0 + ch)
        slot = i % 2
        with torch.cuda.stream(s_in):
            if pin_in:
                a_dev[c0:c1].copy_(a_host[c0:c1], non_blocking=True)
            else:
                st = _staging(device, (ch, k), ("in", slot))
                if i >= 2:
                    ev_in[slot].synchronize()  # the H2D that last read this slot is done
                st[: c1 - c0].copy_(a_host[c0:c1])
                a_dev[c0:c1].copy_(st[: c1 - c0], non_blocking=True)
                ev_in[slot].record(s_in)
            plan.prep(a_dev[c0:c1], Layout.ROW_MAJOR, out=at[:, c0:c1], stream=s_in)
        cur.wait_stream(s_in)
        plan.gemm(at[:, c0:c1], out=ct[:, c0:c1], out_dtype=torch.float32, stream=cur)
        s_out.wait_stream(cur)
        if pin_out:
            _lib.call("tw_copy_2d", buf.ctypes.data + c0 * 4, m * 4, ct.data_ptr() + c0 * 4, m * 4, (c1 - c0) * 4, n, 1,
                      s_out.cuda_stream)
        else:
            drain(slot)  # staging slot free again (its previous chunk copied out)
            so = _staging(device, (n, ch), ("out", slot))
            _lib.call("tw_copy_2d", so.data_ptr(), ch * 4, ct.data_ptr() + c0 * 4, m * 4, (c1 - c0) * 4, n, 1,
                      s_out.cuda_stream)
            ev_out[slot] = torch.cuda.Event()
            ev_out[slot].record(s_out)
            pending[slot] = (c0, c1)
    drain(0)
    drain(1)
    s_out.synchronize()
    cur.wait_stream(s_out)
    a_dev.record_stream(s_in)
    return DenseMatrix(m, n, Layout.COL_MAJOR, buf)


def _device_csc(s: CscMatrix, device) -> DeviceCsc:
    cache = getattr(s, "_tw_b200_dev", None)
    if cache is None:
        cache = {}
        object.__setattr__(s, "_tw_b200_dev", cache)
    if str(device) not in cache:
        cache[str(device)] = DeviceCsc(s, device)
    return cache[str(device)]


def spmm_csc(a: DenseMatrix, s: CscMatrix, *, device=None, out=None) -> DenseMatrix:
    """engine.py:167-181 on the GPU (fp32 activations: bit-exact)."""
    a, s = as_dense(a), as_csc(s)
    if a.cols != s.rows:
        raise DimensionError(f"A has {a.cols} cols but S has {s.rows} rows")
    device = device or torch.device("cuda", torch.cuda.current_device())
    if a.rows == 0:
        return DenseMatrix(0, s.cols, Layout.COL_MAJOR, np.zeros(0, np.float32))
    with torch.cuda.device(device):
        at = _device_activations(a, device, torch.float32)
        ct = spmm_csc_device(at, _device_csc(s, device))
        return _to_host_colmajor(ct, a.rows, s.cols, out)


def gemm_tew(a: DenseMatrix, tiles: CompactTileSet, ew: CscMatrix, workers: int = 1, *, device=None,
             out=None, precision: str | None = None) -> DenseMatrix:
    """engine.py:184-198: gemm_tw + spmm_csc over all N columns.

    precision "fp32" / "exact" keep the reference's composition exactly: the
    TW product (this precision's gemm_tw, bit-identical to it) and the CSC
    SpMM on fp32 activations (bit-identical to spmm_csc), summed with one
    fp32 addition per element (engine.py:197) -- so gemm_tew == gemm_tw +
    spmm_csc bit for bit (test_acceptance.py:84-120).  "bf16" runs the
    overlay folded into one TW plan on the tensor cores (TwPlan.gemm_tew)."""
    a, ew = as_dense(a), as_csc(ew)
    tiles = _as_tileset(tiles)
    if ew.rows != tiles.k or ew.cols != tiles.n:
        raise DimensionError(f"overlay is {ew.rows}x{ew.cols}, pattern is {tiles.k}x{tiles.n}")
    if a.cols != tiles.k:
        raise DimensionError(f"A has {a.cols} cols but pattern K is {tiles.k}")
    _check_workers(workers)
    precision = _precision(precision)
    if ew.nnz == 0:
        return gemm_tw(a, tiles, workers, device=device, out=out, precision=precision)  # engine.py:194-195
    device = device or torch.device("cuda", torch.cuda.current_device())
    if a.rows == 0:
        return DenseMatrix(0, tiles.n, Layout.COL_MAJOR, np.zeros(0, np.float32))
    plan = _plan_for(tiles, device, precision)
    with torch.cuda.device(device):
        a32 = _device_fp32(a, device)
        if precision == "bf16":
            ct = plan.gemm_tew(plan.prep(a32, a.layout), _device_csc(ew, device), out_dtype=torch.float32)
        else:
            ct = plan.gemm(plan.prep(a32, a.layout), out_dtype=torch.float32)
            spmm_csc_device(prep_activations(a32, a.layout, torch.float32), _device_csc(ew, device), out=ct,
                            accumulate=True)
        return _to_host_colmajor(ct, a.rows, tiles.n, out)


def gemm_dense(a: DenseMatrix, b: DenseMatrix, *, device=None, precision: str | None = None) -> DenseMatrix:
    """matrix.py:149-166 through the same kernel: a dense pattern (nothing
    pruned, G = 128) is an ordinary GEMM."""
    a, b = as_dense(a), as_dense(b)
    if a.cols != b.rows:
        raise DimensionError(f"A is {a.shape}, B is {b.shape}: inner dims differ")
    return gemm_tw(a, compact(b, dense_pattern(b.rows, b.cols, 128)), device=device, precision=precision)


# ------------------------------------------------------------------ the reference engine's task API

@dataclass(frozen=True)
class TileTask:
    """engine.py:24-37: one tile's sub-GEMM -- gathered A^T rows (k_i x M),
    the compact sub-matrix (k_i x n_i) and its global output columns."""

    index: int
    gathered_at: np.ndarray
    b_sub: np.ndarray
    out_rows: np.ndarray

    @property
    def flops(self) -> int:
        return 2 * int(self.gathered_at.shape[1]) * int(self.b_sub.shape[0]) * int(self.b_sub.shape[1])


@dataclass(frozen=True)
class BatchGroup:
    """engine.py:40-50: tasks of equal tile width n_i."""

    n_i: int
    tasks: tuple

    @property
    def flops(self) -> int:
        return sum(t.flops for t in self.tasks)


def gather_rows(at, row_mask_words, force_copy: bool = False):
    """engine.py:61-69: the kept rows of A^T (K x M) in original order; a
    full mask returns `at` itself unless force_copy.  numpy in -> numpy out;
    a CUDA tensor in -> one device gather (index_select) out."""
    k = at.shape[0]
    keep = unpack_mask_words(np.asarray(row_mask_words, np.uint32), k).astype(bool)
    if keep.all():
        return at.clone() if (force_copy and torch is not None and isinstance(at, torch.Tensor)) else (
            at.copy() if force_copy else at)
    idx = np.flatnonzero(keep)
    if torch is not None and isinstance(at, torch.Tensor):
        return at.index_select(0, torch.from_numpy(idx).to(at.device)).contiguous()
    return np.ascontiguousarray(at[idx])


def group_by_shape(tasks) -> list:
    """engine.py:72-81: groups of equal n_i (the reference keys on n_i only,
    SURVEY finding 3), largest total FLOPs first, ties by first task index."""
    by_width: dict = {}
    for t in tasks:
        by_width.setdefault(int(t.b_sub.shape[1]), []).append(t)
    groups = [BatchGroup(w, tuple(ts)) for w, ts in by_width.items()]
    groups.sort(key=lambda gr: (-gr.flops, gr.tasks[0].index))
    return groups


def execute_batched(groups, n: int, workers: int = 1, *, device=None, precision: str | None = None) -> np.ndarray:
    """engine.py:84-123: run every task into one (N, M) transposed output
    (zeros where no task writes).  On B200 the whole task list is ONE
    persistent TW-GEMM launch: the tasks' gathered A^T blocks are stacked
    into one operand (sum k_i x M) and task t becomes a tile whose kept rows
    are its own block -- the LPT bins of the reference's thread pool become
    the kernel's static CTA schedule.  Disjoint output rows, fixed per-element
    accumulation order: the result does not depend on `workers` (accepted for
    signature parity)."""
    if workers < 1:
        raise DimensionError(f"workers must be >= 1, got {workers}")
    if n < 1:
        raise DimensionError(f"output needs n >= 1, got {n}")
    tasks = [t for g in groups for t in g.tasks]
    m = int(tasks[0].gathered_at.shape[1]) if tasks else 1
    if not tasks or m == 0:
        return np.zeros((n, m), dtype=np.float32)
    ks = [int(t.gathered_at.shape[0]) for t in tasks]
    kk = int(sum(ks))
    stacked = np.concatenate([np.asarray(t.gathered_at, np.float32).reshape(k_i, m) for t, k_i in zip(tasks, ks)])
    cover = []
    out_tiles = []
    row0 = 0
    for t, k_i in zip(tasks, ks):
        rows = np.asarray(t.out_rows, np.int64)
        if rows.size and (np.any(np.diff(rows) <= 0) or rows[0] < 0 or rows[-1] >= n):
            raise DimensionError("task out_rows must be strictly ascending column ids < n")
        keep = np.zeros(kk, dtype=bool)
        keep[row0: row0 + k_i] = True
        b = np.asarray(t.b_sub, np.float32).reshape(k_i, rows.size)
        out_tiles.append(CompactTile(sub_matrix=DenseMatrix(k_i, rows.size, Layout.COL_MAJOR,
                                                            np.ascontiguousarray(b.T).reshape(-1)),
                                     row_mask_words=pack_mask_words(keep), col_ids=rows.astype(np.int32)))
        cover.append(rows)
        row0 += k_i
    allc = np.concatenate(cover) if cover else np.zeros(0, np.int64)
    if np.unique(allc).size != allc.size:
        raise DimensionError("tasks write overlapping output columns")
    # tiles in ascending first-column order with width <= G (TilePattern's invariants)
    order = sorted(range(len(out_tiles)), key=lambda i: (int(cover[i][0]) if cover[i].size else n, i))
    g = max([1] + [int(c.size) for c in cover])
    ts = CompactTileSet(kk, n, g, tuple(out_tiles[i] for i in order))
    device = device or torch.device("cuda", torch.cuda.current_device())
    plan = TwPlan(ts, device=device, precision=_precision(precision))
    with torch.cuda.device(device):
        at_dev = torch.from_numpy(np.ascontiguousarray(stacked)).to(device)
        ct = plan.gemm(plan.prep(at_dev, Layout.COL_MAJOR), out_dtype=torch.float32)
        return ct.cpu().numpy()


def flop_report(tiles: CompactTileSet, m: int, wall_time: float) -> FlopReport:
    """engine.py:201-209"""
    if m < 1:
        raise DimensionError(f"M must be >= 1, got {m}")
    flops = sum(2 * m * t.sub_matrix.rows * t.sub_matrix.cols for t in tiles.tiles)
    dense = 2 * m * tiles.k * tiles.n
    return FlopReport(wall_time=wall_time, flops=flops, dense_flops=dense, ratio=flops / dense)


def time_median(fn, repeats: int, warmup: int = 1) -> tuple:
    """engine.py:212-223 (wall clock, monotonic).  For device timing use
    CUDA events (bench.py)."""
    for _ in range(warmup):
        fn()
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    arr = np.asarray(times)
    return float(np.median(arr)), float(arr.mean()), float(arr.std())
