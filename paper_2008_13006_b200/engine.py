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


def _code(dtype) -> int:
    if dtype not in _DT:
        raise ValueError(f"unsupported dtype {dtype}; use float32, bfloat16 or float16")
    return _DT[dtype]


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
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


class PackedPlan:
    """The packed image of a CompactTileSet (csrc/tw_pack.cpp): padded kept-K
    index lists, output column ids, the zero-row list (pruned columns and
    dead tiles) and the swizzled 16-bit weight image.  Host-only: built and
    inspected on any machine (tw_plan_build_host)."""

    _create = "tw_plan_build_host"

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
        ranges.  Host-side; returns (units[n,4], unit_off[G+1], zero_off[G+1])."""
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


class TwPlan(PackedPlan):
    """A CompactTileSet packed for the persistent kernel and resident on one
    GPU (see PackedPlan for the layout).

    col_range=(c0, c1) builds a shard that computes output columns [c0, c1)
    only (rows re-based to 0) -- the unit of the N-sharded multi-GPU path.
    """

    _create = "tw_plan_create"

    def __init__(self, tiles: CompactTileSet, device=None, dtype=None, col_range=None, _arrays=None):
        if torch is None:
            raise RuntimeError("torch is required for device plans")
        dtype = dtype or torch.bfloat16
        if dtype not in (torch.bfloat16, torch.float16):
            raise ValueError("plan dtype must be bfloat16 or float16")
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        super().__init__(tiles, "bf16" if dtype == torch.bfloat16 else "fp16", col_range, _arrays)

    @classmethod
    def _from_arrays(cls, k, n, g, col_off, col_ids, words, subs, sub_off, device=None, dtype=None, col_range=None):
        return cls(None, device=device, dtype=dtype, col_range=col_range,
                   _arrays=(int(k), int(n), int(g), col_off, col_ids, words, subs, sub_off))

    def _build(self, *args):
        with torch.cuda.device(self.device):
            super()._build(*args)

    # -------------------------------------------------------------- compute
    def _check_at(self, at):
        if not (isinstance(at, torch.Tensor) and at.is_cuda):
            raise TypeError("at must be a CUDA tensor (K x M)")
        if at.dim() != 2 or at.shape[0] != self.k:
            raise DimensionError(f"A^T has {at.shape[0] if at.dim() == 2 else '?'} rows but pattern K is {self.k}")
        if at.dtype != self.dtype:
            raise TypeError(f"activations must be {self.dtype} (plan dtype), got {at.dtype}")
        if at.stride(1) != 1:
            raise ValueError("A^T must be row-contiguous (M contiguous)")
        return at.shape[1], at.stride(0)

    def _out(self, m, out, out_dtype):
        if out is None:
            return torch.empty((self.n_rows, m), dtype=out_dtype, device=self.device)
        if out.shape != (self.n_rows, m) or out.dtype != out_dtype or out.stride(1) != 1:
            raise DimensionError(f"out must be a ({self.n_rows}, {m}) row-contiguous {out_dtype} tensor")
        return out

    def gemm(self, at, out=None, out_dtype=None, accumulate=False, stream=None, bias=None, relu=False,
             write_pruned=True):
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
        m, lda = self._check_at(at)
        if (accumulate or not write_pruned) and out is None:
            raise ValueError("accumulate=True / write_pruned=False need out")
        ct = self._out(m, out, out_dtype)
        flags = (1 if accumulate else 0) | (0 if write_pruned else 2)
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
        _lib.call("tw_gemm_ex", self._h, at.data_ptr(), m, lda, ct.data_ptr(), ct.stride(0), _code(out_dtype),
                  flags, bias_ptr, 1 if relu else 0, _stream_ptr(stream))
        return ct

    def gemm_exact(self, at32, out=None, stream=None):
        """Bit-exact CUDA-core variant (fp32 activations): mm_accum's exact
        multiply/add sequence, for layout/indexing proofs."""
        if at32.dtype != torch.float32 or at32.shape[0] != self.k or at32.stride(1) != 1:
            raise DimensionError("gemm_exact needs fp32 A^T (K x M), row-contiguous")
        m = at32.shape[1]
        ct = self._out(m, out, torch.float32)
        _lib.call("tw_gemm_exact", self._h, at32.data_ptr(), m, at32.stride(0), ct.data_ptr(), ct.stride(0),
                  _stream_ptr(stream))
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
            cache = self.__dict__.setdefault("_tew_plans", {})
            key = id(csc)
            if key not in cache or cache[key][0] is not csc:
                ts = tew_merged_tileset(self._tiles, csc.host)
                cache[key] = (csc, TwPlan(ts, device=self.device, dtype=self.dtype,
                                          col_range=(self.col_begin, self.col_end)))
            return cache[key][1].gemm(at, out=out, out_dtype=out_dtype, stream=stream)
        ct = self._out(m, out, out_dtype)
        _lib.call("tw_gemm_tew", self._h, at.data_ptr(), m, lda, csc.col_ptr.data_ptr(), csc.row_idx.data_ptr(),
                  csc.values.data_ptr(), csc.nnz, ct.data_ptr(), ct.stride(0), _code(out_dtype), _stream_ptr(stream))
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
              _code(out.dtype), 1 if accumulate else 0, _stream_ptr(stream))
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
              _code(dtype), _stream_ptr(stream))
    return out


# ------------------------------------------------------------------ reference-signature API

def _plan_for(tiles: CompactTileSet, device) -> TwPlan:
    cache = getattr(tiles, "_tw_b200_plans", None)
    if cache is None:
        cache = {}
        object.__setattr__(tiles, "_tw_b200_plans", cache)
    key = str(device)
    if key not in cache:
        cache[key] = TwPlan(tiles, device=device)
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


def _device_activations(a: DenseMatrix, device, dtype):
    """Host DenseMatrix -> device A^T (K x M) in `dtype`.  The fp32 buffer is
    copied as-is (asynchronously when it lives in pinned memory) and
    transposed / cast on the device by the prep kernel."""
    data = np.asarray(a.data, np.float32)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # frozen (read-only) buffers are only read here
        host = torch.from_numpy(data)
    dev = host.to(device, non_blocking=host.is_pinned())
    if a.layout == Layout.ROW_MAJOR:
        return prep_activations(dev.view(a.rows, a.cols), Layout.ROW_MAJOR, dtype)
    return prep_activations(dev.view(a.cols, a.rows), Layout.COL_MAJOR, dtype)


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


def gemm_tw(a: DenseMatrix, tiles: CompactTileSet, workers: int = 1, *, device=None, out=None) -> DenseMatrix:
    """engine.py:152-164: C = A x expand(tiles) as a COL_MAJOR DenseMatrix.
    Pruned columns are exactly zero.  Computes on the GPU with bf16 operands
    and fp32 accumulation/output.  `out`: optional float32 host array
    (M*N, pinned for full copy bandwidth) that receives the C^T buffer."""
    a = as_dense(a)
    tiles = _as_tileset(tiles)
    if a.cols != tiles.k:
        raise DimensionError(f"A has {a.cols} cols but pattern K is {tiles.k}")
    _check_workers(workers)
    device = device or torch.device("cuda", torch.cuda.current_device())
    if a.rows == 0:
        return DenseMatrix(0, tiles.n, Layout.COL_MAJOR, np.zeros(0, np.float32))
    plan = _plan_for(tiles, device)
    if a.layout == Layout.ROW_MAJOR and a.rows >= 2 * _PIPE_CHUNK and _PIPE_ON:
        return _gemm_tw_pipelined(a, plan, device, out)
    at = _device_activations(a, device, plan.dtype)
    ct = plan.gemm(at, out_dtype=torch.float32)
    return _to_host_colmajor(ct, a.rows, tiles.n, out)


_PIPE_CHUNK = int(os.environ.get("TW_B200_PIPE_CHUNK", "1024"))
_PIPE_ON = os.environ.get("TW_B200_PIPE", "1") != "0"
_pipe_streams: dict = {}


def _gemm_tw_pipelined(a: DenseMatrix, plan: "TwPlan", device, out=None) -> DenseMatrix:
    """gemm_tw's host round trip in token chunks on three streams: the H2D
    copy + transpose/cast of chunk c+1, the TW-GEMM of chunk c and the 2-D
    D2H copy of C^T's columns for chunk c-1 overlap (PCIe is full duplex).
    Every chunk is the same kernel on a token slice (A^T columns / C^T
    columns with the full row pitch), so the result is identical to the
    one-shot path."""
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
    a_dev = torch.empty((m, k), dtype=torch.float32, device=device)
    ld = (m + 7) // 8 * 8
    at = torch.empty((k, ld), dtype=plan.dtype, device=device)[:, :m]
    ct = torch.empty((n, m), dtype=torch.float32, device=device)
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    pinned = a_host.is_pinned()
    for c0 in range(0, m, _PIPE_CHUNK):
        c1 = min(m, c0 + _PIPE_CHUNK)
        with torch.cuda.stream(s_in):
            a_dev[c0:c1].copy_(a_host[c0:c1], non_blocking=pinned)
            prep_activations(a_dev[c0:c1], Layout.ROW_MAJOR, plan.dtype, out=at[:, c0:c1], stream=s_in)
        cur.wait_stream(s_in)
        plan.gemm(at[:, c0:c1], out=ct[:, c0:c1], out_dtype=torch.float32, stream=cur)
        s_out.wait_stream(cur)
        _lib.call("tw_copy_2d", buf.ctypes.data + c0 * 4, m * 4, ct.data_ptr() + c0 * 4, m * 4, (c1 - c0) * 4, n, 1,
                  s_out.cuda_stream)
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
    at = _device_activations(a, device, torch.float32)
    ct = spmm_csc_device(at, _device_csc(s, device))
    return _to_host_colmajor(ct, a.rows, s.cols, out)


def gemm_tew(a: DenseMatrix, tiles: CompactTileSet, ew: CscMatrix, workers: int = 1, *, device=None,
             out=None) -> DenseMatrix:
    """engine.py:184-198: gemm_tw + spmm_csc over all N columns."""
    a, ew = as_dense(a), as_csc(ew)
    tiles = _as_tileset(tiles)
    if ew.rows != tiles.k or ew.cols != tiles.n:
        raise DimensionError(f"overlay is {ew.rows}x{ew.cols}, pattern is {tiles.k}x{tiles.n}")
    if a.cols != tiles.k:
        raise DimensionError(f"A has {a.cols} cols but pattern K is {tiles.k}")
    _check_workers(workers)
    if ew.nnz == 0:
        return gemm_tw(a, tiles, workers, device=device, out=out)
    device = device or torch.device("cuda", torch.cuda.current_device())
    if a.rows == 0:
        return DenseMatrix(0, tiles.n, Layout.COL_MAJOR, np.zeros(0, np.float32))
    plan = _plan_for(tiles, device)
    at = _device_activations(a, device, plan.dtype)
    ct = plan.gemm_tew(at, _device_csc(ew, device), out_dtype=torch.float32)
    return _to_host_colmajor(ct, a.rows, tiles.n, out)


def gemm_dense(a: DenseMatrix, b: DenseMatrix, *, device=None) -> DenseMatrix:
    """matrix.py:149-166 through the same kernel: a dense pattern (nothing
    pruned, G = 128) is an ordinary GEMM."""
    a, b = as_dense(a), as_dense(b)
    if a.cols != b.rows:
        raise DimensionError(f"A is {a.shape}, B is {b.shape}: inner dims differ")
    return gemm_tw(a, compact(b, dense_pattern(b.rows, b.cols, 128)), device=device)


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
