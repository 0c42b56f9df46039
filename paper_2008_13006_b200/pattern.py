"""Tile-sparsity patterns and the host metadata packer (north_star item 1).

Mirrors the reference's `tilewise.pattern` types and functions on the hot
path (pattern.py:34-266, :351-370).  The byte-level work -- mask-word
packing, kept-index lists, compaction and pruned-column lists -- runs in the
C++ packer of libtw_b200.so (csrc/tw_pack.cpp), bit-exact with the
reference (tests/test_packer.py pins it against the golden fixtures).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .matrix import DenseMatrix, DimensionError, Layout, as_dense

MASK_WORD_BITS = 32


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def exact_count(fraction: float, total: int) -> int:
    """pattern.py:34-39: floor(fraction*total) with a 1e-9 bias."""
    return int(math.floor(fraction * total + 1e-9))


@dataclass(frozen=True)
class TileConfig:
    """pattern.py:42-57"""
    g: int
    ty: int = 8

    def __post_init__(self) -> None:
        if self.g < 1:
            raise DimensionError(f"granularity must be >= 1, got {self.g}")
        if self.g % 8 != 0:
            raise DimensionError(f"granularity must be a multiple of 8, got {self.g}")
        if self.ty < 1:
            raise DimensionError(f"ty must be >= 1, got {self.ty}")


@dataclass(frozen=True)
class Tile:
    """pattern.py:60-77: sorted global col ids (int32) + per-row keep mask."""
    col_ids: np.ndarray
    row_keep: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "col_ids", np.ascontiguousarray(self.col_ids, dtype=np.int32))
        object.__setattr__(self, "row_keep", np.ascontiguousarray(self.row_keep, dtype=bool))
        self.col_ids.setflags(write=False)
        self.row_keep.setflags(write=False)

    @property
    def k_i(self) -> int:
        return int(np.count_nonzero(self.row_keep))

    @property
    def n_i(self) -> int:
        return int(self.col_ids.size)


@dataclass(frozen=True)
class TilePattern:
    """pattern.py:80-129, with the same invariants and DimensionError messages."""
    k: int
    n: int
    g: int
    tiles: tuple

    def __post_init__(self) -> None:
        object.__setattr__(self, "tiles", tuple(self.tiles))
        if self.k < 1 or self.n < 1 or self.g < 1:
            raise DimensionError(f"bad pattern dims K={self.k} N={self.n} G={self.g}")
        seen = np.concatenate([t.col_ids for t in self.tiles]) if self.tiles else np.empty(0, np.int32)
        if seen.size:
            if seen.min() < 0 or seen.max() >= self.n:
                raise DimensionError("column id out of range")
            if np.unique(seen).size != seen.size:
                raise DimensionError("column ids must be disjoint across tiles")
        for i, t in enumerate(self.tiles):
            if t.row_keep.size != self.k:
                raise DimensionError(f"tile {i} row_keep length {t.row_keep.size} != K={self.k}")
            if t.n_i == 0:
                raise DimensionError(f"tile {i} is empty; empty tiles must be dropped")
            if np.any(np.diff(t.col_ids) <= 0):
                raise DimensionError(f"tile {i} col_ids must be strictly ascending")
            if not (t.n_i == self.g or (i == len(self.tiles) - 1 and t.n_i < self.g)):
                raise DimensionError(
                    f"tile {i} has width {t.n_i}; only the last tile may be narrower than G={self.g}")

    @property
    def surviving_columns(self) -> np.ndarray:
        if not self.tiles:
            return np.empty(0, dtype=np.int32)
        return np.concatenate([t.col_ids for t in self.tiles])

    def keep_mask(self) -> np.ndarray:
        mask = np.zeros((self.k, self.n), dtype=bool)
        for t in self.tiles:
            mask[np.ix_(t.row_keep, t.col_ids)] = True
        return mask

    def unit_counts(self) -> tuple[int, int, int, int]:
        pruned_cols = self.n - int(self.surviving_columns.size)
        total_rows = len(self.tiles) * self.k
        return pruned_cols, self.n, total_rows - sum(t.k_i for t in self.tiles), total_rows


@dataclass(frozen=True)
class CompactTile:
    """pattern.py:132-142: k_i x n_i COL_MAJOR sub-matrix + mask words + col ids."""
    sub_matrix: DenseMatrix
    row_mask_words: np.ndarray
    col_ids: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "row_mask_words", np.ascontiguousarray(self.row_mask_words, dtype=np.uint32))
        object.__setattr__(self, "col_ids", np.ascontiguousarray(self.col_ids, dtype=np.int32))
        self.row_mask_words.setflags(write=False)
        self.col_ids.setflags(write=False)


@dataclass(frozen=True, eq=False)
class CompactTileSet:
    """pattern.py:145-158.  (eq=False: identity-hashable, so device plans can
    be cached per tile set.)"""
    k: int
    n: int
    g: int
    tiles: tuple

    def expand(self) -> DenseMatrix:
        out = np.zeros((self.k, self.n), dtype=np.float32)
        for t in self.tiles:
            rows = mask_words_to_indices(t.row_mask_words, self.k)
            out[np.ix_(rows, t.col_ids)] = t.sub_matrix.array()
        return DenseMatrix.from_array(out, Layout.ROW_MAJOR)


@dataclass(frozen=True)
class PatternStats:
    sparsity: float
    flops: int
    per_tile_dims: tuple
    tiles_dropped: int


# ---------------------------------------------------------------- packer (C ABI)

def pack_mask_words(keep) -> np.ndarray:
    """pattern.py:169-177 (tw_pack_mask_words)."""
    bits = np.ascontiguousarray(keep, dtype=bool).ravel()
    out = np.zeros((bits.size + 31) // 32, dtype=np.uint32)
    _lib.call("tw_pack_mask_words", _ptr(bits.view(np.uint8)), bits.size, _ptr(out))
    return out


def unpack_mask_words(words, length: int) -> np.ndarray:
    """pattern.py:180-185 (tw_unpack_mask_words)."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.zeros(int(length), dtype=np.uint8)
    _lib.call("tw_unpack_mask_words", _ptr(w), w.size, int(length), _ptr(out))
    return out.view(bool)


def mask_words_to_indices(words, length: int) -> np.ndarray:
    """pattern.py:188-189 (tw_mask_words_to_indices)."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.zeros(max(int(length), 1), dtype=np.int64)
    cnt = ctypes.c_int64(0)
    _lib.call("tw_mask_words_to_indices", _ptr(w), w.size, int(length), _ptr(out), ctypes.byref(cnt))
    return out[: cnt.value].copy()


def _flatten_tiles(tiles, k: int):
    """(col_off int64[T+1], col_ids int32, words uint32[T x nwords]) of a
    TilePattern or CompactTileSet."""
    nwords = (k + 31) // 32
    n_t = len(tiles)
    col_off = np.zeros(n_t + 1, np.int64)
    for i, t in enumerate(tiles):
        col_off[i + 1] = col_off[i] + np.asarray(t.col_ids).size
    col_ids = (np.ascontiguousarray(np.concatenate([np.asarray(t.col_ids, np.int32) for t in tiles]), np.int32)
               if n_t else np.zeros(1, np.int32))
    words = np.zeros((max(n_t, 1), nwords), np.uint32)
    for i, t in enumerate(tiles):
        if hasattr(t, "row_mask_words"):
            w = np.asarray(t.row_mask_words, np.uint32)
            if w.size < nwords:
                raise DimensionError(f"mask words cover {w.size * 32} bits, need {k}")
            words[i] = w[:nwords]
        else:
            words[i] = pack_mask_words(t.row_keep)
    return col_off, col_ids, words


def compact(b: DenseMatrix, p: TilePattern) -> CompactTileSet:
    """pattern.py:223-241 (tw_compact): physically remove pruned rows and
    columns per tile; sub-matrices COL_MAJOR."""
    b = as_dense(b)
    if (b.rows, b.cols) != (p.k, p.n):
        raise DimensionError(f"matrix {b.shape} does not match pattern ({p.k}, {p.n})")
    col_off, col_ids, words = _flatten_tiles(p.tiles, p.k)
    total = sum(t.k_i * t.n_i for t in p.tiles)
    subs = np.zeros(max(total, 1), np.float32)
    sub_off = np.zeros(len(p.tiles) + 1, np.int64)
    data = np.ascontiguousarray(b.data, np.float32)
    _lib.call("tw_compact", _ptr(data), p.k, p.n, int(b.layout), len(p.tiles), _ptr(col_off), _ptr(col_ids),
              _ptr(words), _ptr(subs), _ptr(sub_off))
    tiles = []
    for i, t in enumerate(p.tiles):
        k_i, n_i = t.k_i, t.n_i
        buf = subs[sub_off[i]: sub_off[i + 1]].copy()
        tiles.append(CompactTile(sub_matrix=DenseMatrix(k_i, n_i, Layout.COL_MAJOR, buf),
                                 row_mask_words=words[i].copy(), col_ids=t.col_ids))
    return CompactTileSet(p.k, p.n, p.g, tuple(tiles))


def pruned_columns(p) -> np.ndarray:
    """pruning.py:257-258 _pruned_columns_of (tw_pruned_columns): ascending
    output columns owned by no tile -- the rows of C^T that are exact zeros."""
    k = p.k
    col_off, col_ids, _ = _flatten_tiles(p.tiles, k) if p.tiles else (np.zeros(1, np.int64), np.zeros(1, np.int32), None)
    out = np.zeros(max(p.n, 1), np.int64)
    cnt = ctypes.c_int64(0)
    _lib.call("tw_pruned_columns", p.n, len(p.tiles), _ptr(col_off), _ptr(col_ids), _ptr(out), ctypes.byref(cnt))
    return out[: cnt.value].copy()


# ---------------------------------------------------------------- pattern helpers

def partition(n: int, g: int) -> list:
    """pattern.py:192-197"""
    if n < 1 or g < 1:
        raise DimensionError(f"need N >= 1 and G >= 1, got N={n} G={g}")
    return [(s, min(s + g, n)) for s in range(0, n, g)]


def reorganize_columns(survivors, g: int) -> list:
    """pattern.py:200-211"""
    if g < 1:
        raise DimensionError(f"G must be >= 1, got {g}")
    parts = [np.asarray(s, dtype=np.int32) for s in survivors]
    merged = np.sort(np.concatenate(parts) if parts else np.empty(0, np.int32))
    if merged.size and np.unique(merged).size != merged.size:
        raise DimensionError("survivor lists must be disjoint")
    return [merged[i: i + g] for i in range(0, merged.size, g)]


def dense_pattern(k: int, n: int, g: int) -> TilePattern:
    """pattern.py:214-220"""
    return TilePattern(k, n, g, tuple(Tile(np.arange(a, b, dtype=np.int32), np.ones(k, dtype=bool))
                                      for a, b in partition(n, g)))


def zero_fill(b: DenseMatrix, p: TilePattern) -> DenseMatrix:
    """pattern.py:244-250"""
    b = as_dense(b)
    if (b.rows, b.cols) != (p.k, p.n):
        raise DimensionError(f"matrix {b.shape} does not match pattern ({p.k}, {p.n})")
    return DenseMatrix.from_array(np.where(p.keep_mask(), b.array(), np.float32(0.0)).astype(np.float32),
                                  Layout.ROW_MAJOR)


def pattern_stats(p: TilePattern, m: int) -> PatternStats:
    """pattern.py:253-266"""
    if m < 1:
        raise DimensionError(f"M must be >= 1, got {m}")
    dims = tuple((t.k_i, t.n_i) for t in p.tiles)
    kept = sum(a * b for a, b in dims)
    return PatternStats(sparsity=1.0 - kept / (p.k * p.n), flops=2 * m * kept, per_tile_dims=dims,
                        tiles_dropped=(p.n + p.g - 1) // p.g - len(p.tiles))


def random_uniform_pattern(k: int, n: int, g: int, sparsity: float, seed: int) -> TilePattern:
    """pattern.py:351-370: prune u = 1 - sqrt(1-s) of the columns and of every
    tile's rows; identical RNG draw order, hence the identical pattern."""
    if not 0.0 <= sparsity < 1.0:
        raise DimensionError(f"sparsity must be in [0, 1), got {sparsity}")
    rng = np.random.default_rng(seed)
    u = 1.0 - (1.0 - sparsity) ** 0.5
    keep_cols = np.setdiff1d(np.arange(n, dtype=np.int32),
                             rng.choice(n, size=exact_count(u, n), replace=False))
    pruned_rows = exact_count(u, k)
    tiles = []
    for cols in reorganize_columns([keep_cols], g):
        keep = np.ones(k, dtype=bool)
        keep[rng.choice(k, size=pruned_rows, replace=False)] = False
        tiles.append(Tile(cols, keep))
    return TilePattern(k, n, g, tuple(tiles))
