"""The step before the TW path on the GPU: one pruning stage
(`prune_stage`, pruning.py:262-335) -- SURVEY §8(f) row 4.

The unit scores (column means of the score map, then per-tile row means over
each tile's surviving columns) are computed by CUDA kernels
(`tw_prune_col_means`, `tw_prune_row_means`) in numpy's exact summation
order, so they are bit-identical to the reference's float64 means.  The
exact-count selections (`_select_units`, pruning.py:205-239) are small host
sorts and are restated here with the reference's tie-breaking (ascending
score, then unit index; forced units first, protected units never).  The
result is the same TilePattern the reference returns (tests/test_prune.py
against fixtures written by the reference).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .matrix import ConfigError, DimensionError, as_dense
from .pattern import Tile, TilePattern, exact_count, reorganize_columns

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

NEVER_PRUNE = np.inf  # pruning.py:21


def _scores_array(scores) -> np.ndarray:
    s = scores.scores if hasattr(scores, "scores") else scores
    s = np.ascontiguousarray(s, dtype=np.float64)
    if s.ndim != 2:
        raise DimensionError(f"scores must be 2-D, got ndim={s.ndim}")
    if s.size and s.min() < 0:
        raise DimensionError("scores must be nonnegative")
    return s


def select_units(scores: np.ndarray, budget: int, forced, protected) -> np.ndarray:
    """pruning.py:205-239 (`_select_units`, no pooled tie matrix): `budget`
    unit indices to prune -- all of `forced` first (ascending, clipped to the
    budget), the rest by ascending (score, index) skipping `protected`."""
    n = scores.size
    forced = np.asarray(forced, dtype=np.int64)
    protected = np.asarray(protected, dtype=np.int64)
    if budget > n - protected.size:
        raise ConfigError(f"budget {budget} cannot be met with {protected.size} protected of {n} units")
    take = forced[:budget]
    remaining = budget - take.size
    if remaining == 0:
        return np.sort(take)
    blocked = np.zeros(n, dtype=bool)
    blocked[take] = True
    blocked[protected] = True
    order = np.argsort(scores, kind="stable")
    fill = order[~blocked[order]][:remaining]
    return np.sort(np.concatenate([take, fill]))


def _pruned_columns_of(p: TilePattern) -> np.ndarray:
    surv = np.concatenate([t.col_ids for t in p.tiles]).astype(np.int64) if p.tiles else np.empty(0, np.int64)
    return np.setdiff1d(np.arange(p.n, dtype=np.int64), surv)


def _keep_mask(p: TilePattern) -> np.ndarray:
    mask = np.zeros((p.k, p.n), dtype=bool)
    for t in p.tiles:
        mask[np.ix_(np.asarray(t.row_keep, bool), np.asarray(t.col_ids, np.int64))] = True
    return mask


class _GpuMeans:
    """The score reductions on the GPU (tw_prune_col_means / _row_means)."""

    def __init__(self, s: np.ndarray, device):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.k, self.n = s.shape
        self.s = torch.from_numpy(s).to(self.device)
        self.stream = torch.cuda.current_stream(self.device).cuda_stream

    def cols(self) -> np.ndarray:
        out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        _lib.call("tw_prune_col_means", self.s.data_ptr(), self.k, self.n, out.data_ptr(), self.stream)
        return out.cpu().numpy()

    def rows(self, cols: np.ndarray, off: np.ndarray) -> np.ndarray:
        n_tiles = off.size - 1
        cols_d = torch.from_numpy(np.ascontiguousarray(cols, np.int32)).to(self.device)
        off_d = torch.from_numpy(np.ascontiguousarray(off, np.int64)).to(self.device)
        out = torch.empty(n_tiles * self.k, dtype=torch.float64, device=self.device)
        _lib.call("tw_prune_row_means", self.s.data_ptr(), self.k, self.n, cols_d.data_ptr(), off_d.data_ptr(),
                  n_tiles, out.data_ptr(), self.stream)
        return out.cpu().numpy()


def prune_stage(w, scores, s_t: float, g: int, apriori=None, prev: Optional[TilePattern] = None, *,
                device=None, _means=None) -> TilePattern:
    """pruning.py:262-335 with the score reductions on the GPU.  `w` fixes the
    shape (DenseMatrix or array), `scores` is a ScoreMap (or a K x N float64
    array), `apriori` a duck-typed AprioriConfig (ew_reference,
    forced_and_protected()), `prev` the previous stage's pattern.  (`_means`:
    test hook replacing the GPU reductions.)"""
    w = as_dense(w) if not isinstance(w, np.ndarray) else w
    shape = (w.rows, w.cols) if hasattr(w, "rows") else tuple(w.shape)
    s = _scores_array(scores)
    if shape != s.shape:
        raise DimensionError(f"weight {shape} and scores {s.shape} differ")
    if not 0.0 <= s_t < 1.0:
        raise ConfigError(f"s_t must be in [0, 1), got {s_t}")
    k, n = shape
    col_budget = exact_count(s_t, n)
    forced_cols = np.empty(0, dtype=np.int64)
    prev_keep = None
    if prev is not None:
        if (prev.k, prev.n) != (k, n):
            raise DimensionError("previous pattern shape does not match")
        forced_cols = _pruned_columns_of(prev)
        if forced_cols.size > col_budget:
            raise ConfigError(f"s_t regression: {forced_cols.size} columns already pruned, budget {col_budget}")
        prev_keep = _keep_mask(prev)

    means = _means(s) if _means is not None else _GpuMeans(s, device)
    col_scores = means.cols()

    protected = np.empty(0, dtype=np.int64)
    if apriori is not None:  # apriori_tuning, pruning.py:242-254 / :295-304
        if col_scores.size != np.asarray(apriori.ew_reference).size:
            raise DimensionError(f"{col_scores.size} unit scores vs {np.asarray(apriori.ew_reference).size} "
                                 "reference entries")
        ap_forced, protected = apriori.forced_and_protected()
        ap_forced = np.asarray(ap_forced, np.int64)
        protected = np.asarray(protected, np.int64)
        col_scores = col_scores.copy()
        col_scores[ap_forced] = 0.0
        col_scores[protected] = NEVER_PRUNE
        if np.intersect1d(ap_forced, protected).size or np.intersect1d(forced_cols, protected).size:
            raise ConfigError("apriori protection conflicts with forced prunes")
        forced_cols = np.union1d(forced_cols, ap_forced)
        if forced_cols.size > col_budget:
            raise ConfigError(f"{forced_cols.size} forced column prunes exceed budget {col_budget}")
    pruned_cols = select_units(col_scores, col_budget, forced_cols, protected)

    keep_cols = np.setdiff1d(np.arange(n, dtype=np.int64), pruned_cols)
    col_groups = reorganize_columns([keep_cols], g)
    ntiles = len(col_groups)
    if ntiles == 0:
        return TilePattern(k, n, g, ())

    # row phase: unit (t, r) = t*K + r, score = mean over the tile's columns
    cols = np.ascontiguousarray(np.concatenate(col_groups), np.int32)
    off = np.zeros(ntiles + 1, np.int64)
    off[1:] = np.cumsum([c.size for c in col_groups])
    row_score = means.rows(cols, off)
    row_budget = exact_count(s_t, ntiles * k)
    forced_rows = np.empty(0, dtype=np.int64)
    if prev_keep is not None:
        dead = [np.flatnonzero(~prev_keep[:, c.astype(np.int64)].any(axis=1)) + t * k
                for t, c in enumerate(col_groups)]
        forced_rows = np.concatenate(dead) if dead else forced_rows
    pruned_rows = select_units(row_score, row_budget, forced_rows, np.empty(0, np.int64))

    pruned_set = np.zeros(ntiles * k, dtype=bool)
    pruned_set[pruned_rows] = True
    tiles = [Tile(c.astype(np.int32), ~pruned_set[t * k:(t + 1) * k]) for t, c in enumerate(col_groups)]
    return TilePattern(k, n, g, tuple(tiles))


# ---------------------------------------------------------------- TEW overlay
# The input definition of the TEW path (gemm_tew): which pruned weights come
# back as an element-wise CSC overlay.  pruning.py:132-144 (TewConfig),
# :147-159 (score maps), :527-561 (tew_overlay).

@dataclass(frozen=True)
class ScoreMap:
    """Per-element importance scores (K x N, float64, nonnegative, frozen) --
    pruning.py:28-47."""

    scores: np.ndarray

    def __post_init__(self) -> None:
        s = _scores_array(self.scores)
        object.__setattr__(self, "scores", s)
        s.setflags(write=False)

    @property
    def shape(self) -> tuple:
        return self.scores.shape


def magnitude_scores(w) -> ScoreMap:
    """|w| in float64 (pruning.py:156-159): the score map when there are no
    gradients."""
    return ScoreMap(np.abs(as_dense(w).array().astype(np.float64)))


@dataclass(frozen=True)
class TewConfig:
    """TW pruning at alpha + delta plus a delta fraction of the pruned
    elements restored element-wise (pruning.py:132-144)."""

    alpha: float
    delta: float

    def __post_init__(self) -> None:
        if not (0.0 <= self.delta < self.alpha + self.delta <= 1.0):
            raise ConfigError(f"need 0 <= delta < alpha+delta <= 1, got alpha={self.alpha} delta={self.delta}")


def _restore_order(scores_flat: np.ndarray, device) -> np.ndarray:
    """Positions of `scores_flat` by descending score, ties by ascending
    position -- the reference's np.lexsort((idx, -s)) order.  On the GPU a
    stable descending sort keeps equal scores in position order, which is
    exactly that tie rule; without CUDA (host-side packing tools) numpy's
    stable argsort of -s gives the same permutation."""
    if torch is not None and torch.cuda.is_available() and scores_flat.size > 0:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        s = torch.from_numpy(np.ascontiguousarray(scores_flat)).to(dev)
        return torch.sort(s, descending=True, stable=True).indices.cpu().numpy()
    return np.argsort(-scores_flat, kind="stable")


def tew_overlay(w, scores, pattern: TilePattern, cfg: TewConfig, tol: float = 0.05, *, device=None):
    """pruning.py:527-561: restore the floor(delta*K*N) highest-scored
    elements the pattern prunes -- in pruned columns too (SURVEY finding 4) --
    as a CSC overlay holding their original values; the pattern is returned
    unchanged.  Raises ConfigError when the pattern's sparsity is not
    alpha + delta within `tol`, or when delta asks for more elements than
    are pruned; DimensionError on shape mismatches."""
    from .matrix import to_csc
    from .pattern import pattern_stats

    w = as_dense(w)
    s = _scores_array(scores)
    if w.shape != s.shape:
        raise DimensionError(f"weight {w.shape} and scores {s.shape} differ")
    if (pattern.k, pattern.n) != w.shape:
        raise DimensionError("pattern does not match weight matrix")
    sparsity = pattern_stats(pattern, m=1).sparsity
    if abs(sparsity - (cfg.alpha + cfg.delta)) > tol:
        raise ConfigError(f"pattern sparsity {sparsity:.4f} is not alpha+delta={cfg.alpha + cfg.delta:.4f} "
                          f"within {tol}")
    count = exact_count(cfg.delta, pattern.k * pattern.n)
    pruned_flat = np.flatnonzero(~_keep_mask(pattern).ravel())
    if count > pruned_flat.size:
        raise ConfigError(f"delta asks to restore {count} elements but only {pruned_flat.size} are pruned")
    chosen = pruned_flat[_restore_order(s.ravel()[pruned_flat], device)[:count]]
    restore = np.zeros(pattern.k * pattern.n, dtype=bool)
    restore[chosen] = True
    return pattern, to_csc(w, restore.reshape(pattern.k, pattern.n))
