"""N-dimension (column-tile) sharding of one TW layer across the GPUs of a
box -- north_star item 4, SURVEY.md §8(e).

The reference has no distributed code; its only parallelism is the thread
pool over tile groups whose output columns are disjoint (engine.py:4-7,
:89-123).  The same property shards the layer across GPUs with no data-path
collective: rank r owns the contiguous output-column range
[r*P_n, min(N, (r+1)*P_n)), P_n = ceil(N / world), holds only the tiles (or
tile pieces -- a tile straddling a boundary is split by the packer, keeping
its kept-K list) of that range, and computes those C^T rows, zero rows for
pruned columns included.  The one exchange step is reassembling C^T: an
all-gather of equal (P_n x M) row blocks whose receive buffer *is* the full
C^T (row-major N x M, the reference's COL_MAJOR C buffer, engine.py:164), so
no post-scatter is needed.

One process per GPU; the process group is torch.distributed's (NCCL over
NVLink/NVSwitch on a B200 box, gloo for the CPU tests of the host logic).
"""

from __future__ import annotations

import numpy as np

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None

from .engine import TwPlan
from .matrix import DimensionError
from .pattern import CompactTileSet


def shard_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """Equal contiguous output-column ranges, one per rank (the last ones may
    be shorter or empty when world does not divide N)."""
    if n < 0 or world < 1:
        raise DimensionError(f"bad shard request: N={n}, world={world}")
    per = -(-n // world) if n else 0
    return [(min(n, r * per), min(n, (r + 1) * per)) for r in range(world)]


def rows_per_rank(n: int, world: int) -> int:
    return -(-n // world) if n else 0


def _group_info(group):
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def all_gather_rows(local, n: int, group=None, out=None):
    """Reassemble C^T (n x M) from every rank's (rows_per_rank x M) block.

    `local` holds this rank's rows first (rows past its range are padding and
    are dropped).  Returns `out[:n]` -- a contiguous view of the gather
    buffer, so the caller can keep `out` resident across calls."""
    rank, world = _group_info(group)
    per = rows_per_rank(n, world)
    if local.dim() != 2 or local.shape[0] != per:
        raise DimensionError(f"local block must have {per} rows, got {tuple(local.shape)}")
    m = local.shape[1]
    if out is None:
        out = torch.empty((per * world, m), dtype=local.dtype, device=local.device)
    elif out.shape != (per * world, m) or out.dtype != local.dtype or not out.is_contiguous():
        raise DimensionError(f"gather buffer must be a contiguous ({per * world}, {m}) {local.dtype} tensor")
    if world == 1:
        if out.data_ptr() != local.data_ptr():
            out.copy_(local)
    elif local.is_cuda and dist.get_backend(group) != "nccl":
        # gloo (host-logic tests, several ranks per device): stage via the host
        host = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(host, local.contiguous().cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out[:n]


class ShardedTwPlan:
    """One rank's share of an N-sharded TW layer.

    gemm_local(at) computes this rank's C^T rows (no communication); gemm(at)
    also all-gathers the full C^T.  The local block always has
    rows_per_rank(N, world) rows: rows past the rank's range (only on the
    last ranks when world does not divide N) are zero."""

    def __init__(self, tiles: CompactTileSet, group=None, device=None, dtype=None):
        self.group = group
        self.rank, self.world = _group_info(group)
        self.k, self.n = int(tiles.k), int(tiles.n)
        self.ranges = shard_ranges(self.n, self.world)
        self.col_range = self.ranges[self.rank]
        self.per = rows_per_rank(self.n, self.world)
        self.plan = TwPlan(tiles, device=device, dtype=dtype, col_range=self.col_range)
        self.device = self.plan.device
        self._bufs: dict = {}

    @property
    def info(self):
        return self.plan.info

    def _buffers(self, m: int, out_dtype):
        key = (m, out_dtype)
        if key not in self._bufs:
            local = torch.zeros((self.per, m), dtype=out_dtype, device=self.device)
            full = torch.empty((self.per * self.world, m), dtype=out_dtype, device=self.device)
            self._bufs[key] = (local, full)
        return self._bufs[key]

    def gemm_local(self, at, out_dtype=None, stream=None):
        """This rank's C^T rows [c0, c1) (re-based to 0), padded to `per` rows."""
        out_dtype = out_dtype or torch.float32
        m = at.shape[1]
        local, _ = self._buffers(m, out_dtype)
        width = self.col_range[1] - self.col_range[0]
        if width:
            self.plan.gemm(at, out=local[:width], out_dtype=out_dtype, stream=stream)
        return local

    def gemm(self, at, out_dtype=None, stream=None):
        """Full C^T (N x M) on every rank: local TW-GEMM + all-gather."""
        local = self.gemm_local(at, out_dtype, stream)
        _, full = self._buffers(at.shape[1], local.dtype)
        return all_gather_rows(local, self.n, self.group, out=full)


def shard_table(n: int, world: int) -> np.ndarray:
    """(world, 2) int64 array of the shard ranges (for logs and tests)."""
    return np.asarray(shard_ranges(n, world), np.int64).reshape(world, 2)
