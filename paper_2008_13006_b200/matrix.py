"""Host-side matrix types of the drop-in API.

Same names, fields, layout tags and error behaviour as the reference's
`tilewise.matrix` (matrix.py:29-204) so code written against the reference
runs unchanged; the compute behind them is libtw_b200.so.  Objects from the
reference package are accepted wherever these are (duck typing on
rows / cols / layout / data and col_ptr / row_idx / values).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum
from typing import Callable, Union

import numpy as np


class Layout(IntEnum):
    """matrix.py:29-31"""
    ROW_MAJOR = 0
    COL_MAJOR = 1


class DimensionError(ValueError):
    """Operand shapes do not match the operation's contract (matrix.py:34-35)."""


class FormatError(ValueError):
    """A binary file is malformed (matrix.py:38-39)."""


class ConfigError(ValueError):
    """A configuration value is out of range (pruning.py:24-25)."""


@dataclass(frozen=True)
class GemmShape:
    """matrix.py:42-54"""
    m: int
    k: int
    n: int

    def __post_init__(self) -> None:
        if self.m < 1 or self.k < 1 or self.n < 1:
            raise DimensionError(f"GEMM dims must be positive, got {self}")

    @property
    def flops(self) -> int:
        return 2 * self.m * self.k * self.n


@dataclass(frozen=True)
class DenseMatrix:
    """fp32 2-D matrix with a storage-layout tag; the buffer is frozen
    (matrix.py:57-108).  COL_MAJOR storage of C is exactly the C^T buffer the
    engine writes."""

    rows: int
    cols: int
    layout: Layout
    data: np.ndarray

    def __post_init__(self) -> None:
        if self.rows < 0 or self.cols < 0:
            raise DimensionError(f"negative dims {self.rows}x{self.cols}")
        if self.data.dtype != np.float32:
            raise DimensionError(f"buffer must be float32, got {self.data.dtype}")
        if self.data.ndim != 1 or self.data.size != self.rows * self.cols:
            raise DimensionError(f"buffer has {self.data.size} elements, expected {self.rows * self.cols}")
        self.data.setflags(write=False)

    @classmethod
    def from_array(cls, arr, layout: Layout | None = None) -> "DenseMatrix":
        a = np.asarray(arr, dtype=np.float32)
        if a.ndim != 2:
            raise DimensionError(f"expected 2-D array, got ndim={a.ndim}")
        if layout is None:
            layout = Layout.COL_MAJOR if (a.flags.f_contiguous and not a.flags.c_contiguous) else Layout.ROW_MAJOR
        buf = np.ravel(a, order="C" if layout == Layout.ROW_MAJOR else "F")
        if buf.base is not None or np.shares_memory(buf, a):
            buf = buf.copy()  # never alias caller memory (the buffer gets frozen)
        return cls(a.shape[0], a.shape[1], Layout(layout), buf)

    def array(self) -> np.ndarray:
        if self.layout == Layout.ROW_MAJOR:
            return self.data.reshape(self.rows, self.cols)
        return self.data.reshape(self.cols, self.rows).T

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)


@dataclass(frozen=True)
class CscMatrix:
    """Compressed sparse column matrix, fp32 values (matrix.py:111-146)."""

    rows: int
    cols: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        cp = self.col_ptr
        if cp.ndim != 1 or cp.size != self.cols + 1:
            raise DimensionError("col_ptr must have cols+1 entries")
        if cp[0] != 0 or np.any(np.diff(cp.astype(np.int64)) < 0):
            raise FormatError("col_ptr must be nondecreasing and start at 0")
        nnz = int(cp[-1])
        if self.row_idx.size != nnz or self.values.size != nnz:
            raise DimensionError("row_idx/values length must equal col_ptr[-1]")
        if nnz:
            ri = self.row_idx.astype(np.int64)
            if ri.min() < 0 or ri.max() >= self.rows:
                raise DimensionError("row index out of range")
            col_of = np.repeat(np.arange(self.cols), np.diff(cp.astype(np.int64)))
            same = col_of[1:] == col_of[:-1]
            if np.any(np.diff(ri)[same] <= 0):
                raise FormatError("row indices must be strictly increasing per column")
        for name in ("col_ptr", "row_idx", "values"):
            getattr(self, name).setflags(write=False)

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])


def as_dense(a) -> DenseMatrix:
    """Accept this package's DenseMatrix, the reference's, or a 2-D array."""
    if isinstance(a, DenseMatrix):
        return a
    if all(hasattr(a, f) for f in ("rows", "cols", "layout", "data")):
        return DenseMatrix(int(a.rows), int(a.cols), Layout(int(a.layout)),
                           np.asarray(a.data, dtype=np.float32).copy())
    return DenseMatrix.from_array(np.asarray(a, dtype=np.float32))


def as_csc(s) -> CscMatrix:
    """Accept this package's CscMatrix or the reference's (converted once and
    cached on the immutable source object, so device copies and merged TEW
    plans keyed on the converted matrix are reused across calls)."""
    if isinstance(s, CscMatrix):
        return s
    cached = getattr(s, "_tw_b200_csc", None)
    if cached is not None:
        return cached
    out = CscMatrix(int(s.rows), int(s.cols), np.asarray(s.col_ptr, np.uint32).copy(),
                    np.asarray(s.row_idx, np.uint32).copy(), np.asarray(s.values, np.float32).copy())
    try:
        object.__setattr__(s, "_tw_b200_csc", out)
    except Exception:  # objects without a __dict__: convert every call
        pass
    return out


def transpose(m: DenseMatrix) -> DenseMatrix:
    """matrix.py:169-173"""
    return DenseMatrix.from_array(np.ascontiguousarray(as_dense(m).array().T), Layout.ROW_MAJOR)


KeepPredicate = Union[np.ndarray, Callable[[np.ndarray], np.ndarray]]


def to_csc(m: DenseMatrix, keep: KeepPredicate) -> CscMatrix:
    """matrix.py:179-196: CSC of exactly the kept elements, rows ascending."""
    a = as_dense(m).array()
    mask = keep(a) if callable(keep) else np.asarray(keep, dtype=bool)
    if mask.shape != a.shape:
        raise DimensionError(f"keep mask {mask.shape} does not match matrix {a.shape}")
    col, row = np.nonzero(mask.T)
    col_ptr = np.zeros(a.shape[1] + 1, dtype=np.uint32)
    np.cumsum(np.bincount(col, minlength=a.shape[1]), out=col_ptr[1:])
    return CscMatrix(a.shape[0], a.shape[1], col_ptr, row.astype(np.uint32),
                     np.ascontiguousarray(a[row, col], dtype=np.float32))


def csc_to_dense(s: CscMatrix) -> DenseMatrix:
    """matrix.py:199-204"""
    s = as_csc(s)
    out = np.zeros((s.rows, s.cols), dtype=np.float32)
    out[s.row_idx.astype(np.int64), np.repeat(np.arange(s.cols), np.diff(s.col_ptr.astype(np.int64)))] = s.values
    return DenseMatrix.from_array(out, Layout.ROW_MAJOR)
