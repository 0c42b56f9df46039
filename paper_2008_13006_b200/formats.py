"""On-disk formats of the reference, read straight into the packer
(SURVEY.md §8(f) row 2).

Byte layouts (reference pattern.py:373-420,
matrix.py:207-283), all little-endian:

  TWPT  "TWPT" u32 version=1, K, N, G, n_tiles; per tile: u32 n_i,
        u32 col_ids[n_i], u32 row-keep words[ceil(K/32)]
  TWCS  "TWCS" u32 version=1, rows, cols, nnz; u32 col_ptr[cols+1],
        u32 row_idx[nnz], f32 values[nnz]
  TWMX  "TWMX" u32 version=1, rows, cols, u8 layout (0 row-, 1 col-major),
        3 pad bytes; f32 data[rows*cols]

read_/write_ functions mirror the reference's names and FormatError
behaviour (byte-identical output, same rejection of truncated / trailing /
wrong-magic / wrong-version files).  plan_from_files() goes from a TWPT
pattern + TWMX weights to a device-resident TwPlan without building Tile /
CompactTile objects: the parsed column ids and mask words feed the C++
packer (tw_compact + tw_plan_create) directly.
"""

from __future__ import annotations

import struct

import numpy as np

from .matrix import CscMatrix, DenseMatrix, DimensionError, FormatError, Layout
from .pattern import MASK_WORD_BITS, Tile, TilePattern, pack_mask_words, unpack_mask_words

VERSION = 1
_PT = struct.Struct("<IIIII")    # version, K, N, G, n_tiles
_CS = struct.Struct("<IIII")     # version, rows, cols, nnz
_MX = struct.Struct("<IIIB3x")   # version, rows, cols, layout


def _check_magic(raw: bytes, magic: bytes) -> None:
    if raw[:4] != magic:
        raise FormatError(f"bad magic {raw[:4]!r}, expected {magic!r}")


def _header(raw: bytes, st: struct.Struct):
    if len(raw) < 4 + st.size:
        raise FormatError("header truncated")
    vals = st.unpack_from(raw, 4)
    if vals[0] != VERSION:
        raise FormatError(f"unsupported version {vals[0]}")
    return vals[1:]


# ----------------------------------------------------------------- TWPT
def parse_pattern(raw: bytes):
    """TWPT bytes -> (k, n, g, col_off int64[T+1], col_ids int32, words uint32[T*nwords])."""
    _check_magic(raw, b"TWPT")
    k, n, g, ntiles = _header(raw, _PT)
    nwords = (k + MASK_WORD_BITS - 1) // MASK_WORD_BITS
    off = 4 + _PT.size
    col_off = np.zeros(ntiles + 1, np.int64)
    ids, words = [], []
    for t in range(ntiles):
        if len(raw) < off + 4:
            raise FormatError("tile header truncated")
        (n_i,) = struct.unpack_from("<I", raw, off)
        off += 4
        need = 4 * (n_i + nwords)
        if len(raw) < off + need:
            raise FormatError("tile payload truncated")
        ids.append(np.frombuffer(raw, "<u4", n_i, off).astype(np.int32))
        words.append(np.frombuffer(raw, "<u4", nwords, off + 4 * n_i).astype(np.uint32))
        off += need
        col_off[t + 1] = col_off[t] + n_i
    if off != len(raw):
        raise FormatError(f"{len(raw) - off} trailing bytes after last tile")
    col_ids = np.concatenate(ids) if ids else np.zeros(0, np.int32)
    w = np.concatenate(words) if words else np.zeros(0, np.uint32)
    return k, n, g, col_off, col_ids, w


def read_pattern(path) -> TilePattern:
    """pattern.py:385-420 read_pattern."""
    with open(path, "rb") as f:
        raw = f.read()
    k, n, g, col_off, col_ids, words = parse_pattern(raw)
    nwords = (k + MASK_WORD_BITS - 1) // MASK_WORD_BITS
    tiles = [Tile(col_ids[col_off[t]:col_off[t + 1]], unpack_mask_words(words[t * nwords:(t + 1) * nwords], k))
             for t in range(len(col_off) - 1)]
    try:
        return TilePattern(k, n, g, tuple(tiles))
    except DimensionError as e:
        raise FormatError(f"pattern file violates invariants: {e}") from e


def write_pattern(p, path) -> None:
    """pattern.py:376-382 write_pattern (byte-identical)."""
    nwords = (p.k + MASK_WORD_BITS - 1) // MASK_WORD_BITS
    parts = [b"TWPT", _PT.pack(VERSION, p.k, p.n, p.g, len(p.tiles))]
    for t in p.tiles:
        ids = np.asarray(t.col_ids)
        words = pack_mask_words(np.asarray(t.row_keep, bool))
        assert words.size == nwords
        parts += [struct.pack("<I", ids.size), ids.astype("<u4").tobytes(), words.astype("<u4").tobytes()]
    with open(path, "wb") as f:
        f.write(b"".join(parts))


# ----------------------------------------------------------------- TWCS
def read_csc(path) -> CscMatrix:
    """matrix.py:266-283 read_csc."""
    with open(path, "rb") as f:
        raw = f.read()
    _check_magic(raw, b"TWCS")
    rows, cols, nnz = _header(raw, _CS)
    off = 4 + _CS.size
    need = 4 * (cols + 1 + 2 * nnz)
    if len(raw) - off != need:
        raise FormatError(f"payload has {len(raw) - off} bytes, expected {need}")
    col_ptr = np.frombuffer(raw, "<u4", cols + 1, off).astype(np.uint32)
    row_idx = np.frombuffer(raw, "<u4", nnz, off + 4 * (cols + 1)).astype(np.uint32)
    values = np.frombuffer(raw, "<f4", nnz, off + 4 * (cols + 1 + nnz)).astype(np.float32)
    return CscMatrix(rows, cols, col_ptr, row_idx, values)


def write_csc(s, path) -> None:
    """matrix.py:255-263 write_csc (byte-identical)."""
    with open(path, "wb") as f:
        f.write(b"TWCS" + _CS.pack(VERSION, s.rows, s.cols, s.nnz))
        f.write(np.asarray(s.col_ptr).astype("<u4").tobytes())
        f.write(np.asarray(s.row_idx).astype("<u4").tobytes())
        f.write(np.asarray(s.values).astype("<f4").tobytes())


# ----------------------------------------------------------------- TWMX
def read_matrix(path) -> DenseMatrix:
    """matrix.py:219-252 read_matrix (single record)."""
    with open(path, "rb") as f:
        raw = f.read()
    _check_magic(raw, b"TWMX")
    rows, cols, layout = _header(raw, _MX)
    if layout not in (0, 1):
        raise FormatError(f"bad layout byte {layout}")
    if rows == 0 or cols == 0:
        raise FormatError(f"empty matrix {rows}x{cols} in file")
    off = 4 + _MX.size
    need = 4 * rows * cols
    if len(raw) < off + need:
        raise FormatError(f"payload has {len(raw) - off} bytes, expected {need}")
    if len(raw) != off + need:
        raise FormatError(f"{len(raw) - off - need} trailing bytes after payload")
    data = np.frombuffer(raw, "<f4", rows * cols, off).astype(np.float32)
    return DenseMatrix(rows, cols, Layout(layout), data)


def write_matrix(m, path) -> None:
    """matrix.py:211-216 write_matrix (byte-identical)."""
    if m.rows == 0 or m.cols == 0:
        raise FormatError(f"refusing to write empty {m.rows}x{m.cols} matrix")
    with open(path, "wb") as f:
        f.write(b"TWMX" + _MX.pack(VERSION, m.rows, m.cols, int(m.layout)))
        f.write(np.asarray(m.data).astype("<f4").tobytes())


# ----------------------------------------------------------------- packer
def plan_from_files(pattern_path, weights, device=None, dtype=None, col_range=None, host=False):
    """TWPT pattern + weights (TWMX path or DenseMatrix) -> TwPlan on `device`.

    The pattern's parsed arrays go to the C++ packer directly: tw_compact
    (pattern.py:223-241) builds the compacted sub-matrices and tw_plan_create
    packs them, with no per-tile Python objects in between."""
    import ctypes

    from . import _lib
    from .engine import TwPlan

    with open(pattern_path, "rb") as f:
        k, n, g, col_off, col_ids, words = parse_pattern(f.read())
    w = read_matrix(weights) if isinstance(weights, (str, bytes)) or hasattr(weights, "__fspath__") else weights
    if (w.rows, w.cols) != (k, n):
        raise DimensionError(f"weights are {w.rows}x{w.cols}, pattern is {k}x{n}")
    # validate the pattern exactly as TilePattern would (FormatError on violation)
    nwords = (k + MASK_WORD_BITS - 1) // MASK_WORD_BITS
    try:
        TilePattern(k, n, g, tuple(Tile(col_ids[col_off[t]:col_off[t + 1]],
                                        unpack_mask_words(words[t * nwords:(t + 1) * nwords], k))
                                   for t in range(len(col_off) - 1)))
    except DimensionError as e:
        raise FormatError(f"pattern file violates invariants: {e}") from e
    b = np.ascontiguousarray(np.asarray(w.data, np.float32))
    kept = np.array([int(np.unpackbits(words[t * nwords:(t + 1) * nwords].view(np.uint8), bitorder="little")[:k].sum())
                     for t in range(len(col_off) - 1)], np.int64)
    subs = np.zeros(max(1, int((kept * np.diff(col_off)).sum())), np.float32)
    sub_off = np.zeros(len(col_off), np.int64)
    col_off = np.ascontiguousarray(col_off, np.int64)
    col_ids = np.ascontiguousarray(col_ids, np.int32)
    words = np.ascontiguousarray(words, np.uint32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.call("tw_compact", p(b), k, n, int(w.layout), len(col_off) - 1, p(col_off), p(col_ids), p(words), p(subs),
              p(sub_off))
    if host:  # CPU-only packed image (no device buffers), for inspection / tests
        from .engine import PackedPlan
        return PackedPlan._host_from_arrays(k, n, g, col_off, col_ids, words, subs, sub_off, col_range=col_range)
    return TwPlan._from_arrays(k, n, g, col_off, col_ids, words, subs, sub_off, device=device, dtype=dtype,
                               col_range=col_range)


# ----------------------------------------------------------------- TWML
_ML = struct.Struct("<II")  # version, layer count


def _dense_record(raw: bytes, off: int):
    if raw[off:off + 4] != b"TWMX":
        raise FormatError(f"bad magic {raw[off:off + 4]!r}, expected {b'TWMX'!r}")
    if len(raw) < off + 4 + _MX.size:
        raise FormatError("header truncated")
    version, rows, cols, layout = _MX.unpack_from(raw, off + 4)
    if version != VERSION:
        raise FormatError(f"unsupported version {version}")
    if layout not in (0, 1) or rows == 0 or cols == 0:
        raise FormatError(f"bad dense record ({rows}x{cols}, layout {layout})")
    off += 4 + _MX.size
    if len(raw) < off + 4 * rows * cols:
        raise FormatError("dense record truncated")
    m = DenseMatrix(rows, cols, Layout(layout), np.frombuffer(raw, "<f4", rows * cols, off).astype(np.float32))
    return m, off + 4 * rows * cols


def read_model(path):
    """trainer.py:275-306 load_model (TWML checkpoint) -> (weights, biases):
    lists of float32 arrays (K_i x N_i and N_i), for the verify CLI and the
    layer-chaining caller.  (The trainer itself is out of scope.)"""
    with open(path, "rb") as f:
        raw = f.read()
    _check_magic(raw, b"TWML")
    (n_layers,) = _header(raw, _ML)
    off = 4 + _ML.size
    shapes = []
    for _ in range(n_layers):
        if len(raw) < off + 8:
            raise FormatError("shape table truncated")
        shapes.append(struct.unpack_from("<II", raw, off))
        off += 8
    weights, biases = [], []
    for rows, cols in shapes:
        w, off = _dense_record(raw, off)
        if (w.rows, w.cols) != (rows, cols):
            raise FormatError(f"layer blob ({w.rows},{w.cols}) does not match ({rows},{cols})")
        b, off = _dense_record(raw, off)
        if (b.rows, b.cols) != (1, cols):
            raise FormatError(f"bias blob ({b.rows},{b.cols}) does not match (1,{cols})")
        weights.append(w.array().astype(np.float32))
        biases.append(b.array().astype(np.float32).ravel())
    if off != len(raw):
        raise FormatError(f"{len(raw) - off} trailing bytes in checkpoint")
    return weights, biases
