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

import contextlib
import ctypes

import numpy as np

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None

from . import _lib
from .engine import TwPlan, _code, _stream_ptr
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


def cyclic_ranges(n: int, world: int, rounds: int) -> list[list[tuple[int, int]]]:
    """Block-cyclic output-column chunks: chunk c = j*world + r covers
    [c*s, (c+1)*s) (clipped to N), s = ceil(N / (world*rounds)); rank r owns
    chunks r, world + r, 2*world + r, ...  The chunks of round j from all
    ranks are the contiguous rows [j*world*s, (j+1)*world*s) of C^T, so one
    all-gather per round lands every row in place.  rounds=1 is
    shard_ranges."""
    if rounds < 1:
        raise DimensionError(f"rounds must be >= 1, got {rounds}")
    if n < 0 or world < 1:
        raise DimensionError(f"bad shard request: N={n}, world={world}")
    s = -(-n // (world * rounds)) if n else 0
    return [[(min(n, (j * world + r) * s), min(n, (j * world + r + 1) * s)) for j in range(rounds)]
            for r in range(world)]


class ShardedTwPlan:
    """One rank's share of an N-sharded TW layer.

    rounds=1: rank r owns one contiguous column range (shard_ranges).
    rounds=J>1: block-cyclic chunks (cyclic_ranges); gemm() runs round j's
    TW-GEMM, then starts round j's all-gather asynchronously, so NCCL moves
    round j's rows over NVLink while the kernel computes round j+1 --
    SURVEY.md §8(e)'s overlap by chunking.  Every GEMM writes straight into
    its slot of the gather buffer and the all-gather runs in place, so the
    gathered buffer is C^T with no copies.

    gemm_local(at) computes this rank's rows only (no communication) and
    returns them as a (rounds*chunk, M) view stack; rows past N are zero."""

    def __init__(self, tiles: CompactTileSet, group=None, device=None, dtype=None, rounds: int = 1,
                 fused: bool = False):
        self.group = group
        self.rank, self.world = _group_info(group)
        if fused and rounds != 1:
            raise DimensionError("the fused (peer-store) all-gather uses contiguous ranges: rounds must be 1")
        self.fused = bool(fused)
        self._peer: dict = {}
        self.k, self.n = int(tiles.k), int(tiles.n)
        self.rounds = int(rounds)
        self.chunks = cyclic_ranges(self.n, self.world, self.rounds)[self.rank]
        self.chunk = -(-self.n // (self.world * self.rounds)) if self.n else 0
        self.ranges = [r[0] for r in cyclic_ranges(self.n, self.world, 1)] if self.rounds == 1 else None
        self.col_range = self.chunks[0] if self.rounds == 1 else None
        self.per = self.chunk * self.rounds
        self.plans = [TwPlan(tiles, device=device, dtype=dtype, col_range=c) if c[1] > c[0] else None
                      for c in self.chunks]
        self.plan = next((pl for pl in self.plans if pl is not None), None)
        self.device = (self.plan.device if self.plan is not None
                       else torch.device(device) if device is not None
                       else torch.device("cuda", torch.cuda.current_device()))
        self._bufs: dict = {}

    @property
    def info(self):
        return [pl.info if pl is not None else None for pl in self.plans]

    def _full(self, m: int, out_dtype):
        key = (m, out_dtype)
        if key not in self._bufs:
            # rows past N (tail chunks) stay zero: no GEMM ever writes them
            self._bufs[key] = torch.zeros((self.chunk * self.world * self.rounds, m), dtype=out_dtype,
                                          device=self.device)
        return self._bufs[key]

    def _slot(self, full, j):
        c = j * self.world + self.rank
        return full[c * self.chunk:(c + 1) * self.chunk]

    def _compute(self, at, full, j, out_dtype, stream):
        pl, (c0, c1) = self.plans[j], self.chunks[j]
        if pl is not None:
            pl.gemm(at, out=self._slot(full, j)[: c1 - c0], out_dtype=out_dtype, stream=stream)

    def gemm_local(self, at, out_dtype=None, stream=None):
        """This rank's C^T rows, chunk by chunk ((rounds*chunk) x M)."""
        out_dtype = out_dtype or torch.float32
        full = self._full(at.shape[1], out_dtype)
        for j in range(self.rounds):
            self._compute(at, full, j, out_dtype, stream)
        return torch.cat([self._slot(full, j) for j in range(self.rounds)]) if self.rounds > 1 \
            else self._slot(full, 0)

    def _peer_buffers(self, m: int, out_dtype):
        """Fused mode: every rank's full C^T buffer is a CUDA IPC allocation;
        the handles are exchanged once over the process group and opened, so
        this rank's kernel can store its rows into all replicas."""
        key = (m, out_dtype)
        if key in self._peer:
            return self._peer[key]
        esize = torch.tensor([], dtype=out_dtype).element_size()
        rows = self.per * self.world
        nbytes = max(1, rows * m * esize)
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        with torch.cuda.device(self.device):  # allocate / map on the plan's GPU
            _lib.call("tw_ipc_alloc", nbytes, ctypes.byref(ptr), ctypes.cast(handle, ctypes.c_void_p))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        ptrs = []
        for r, h in enumerate(handles):
            if r == self.rank:
                ptrs.append(ptr.value)
            else:
                pp = ctypes.c_void_p()
                hb = (ctypes.c_char * 64).from_buffer_copy(h)
                with torch.cuda.device(self.device):
                    _lib.call("tw_ipc_open", ctypes.cast(hb, ctypes.c_void_p), ctypes.byref(pp))
                ptrs.append(pp.value)
        full = _device_view(ptr.value, (rows, m), out_dtype, self.device)
        full.zero_()  # rows past N stay zero
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        # this rank's rows inside every replica: the local one first
        row0 = self.col_range[0] * m * esize
        order = [self.rank] + [r for r in range(self.world) if r != self.rank]
        dsts = (ctypes.c_void_p * self.world)(*[ptrs[r] + row0 for r in order])
        self._peer[key] = (full, dsts, ptr.value, [ptrs[r] for r in range(self.world) if r != self.rank])
        return self._peer[key]

    def close(self):
        """Release the fused mode's IPC buffers (after a barrier: peers may
        still be storing into this rank's replica otherwise)."""
        if self._peer and dist is not None and dist.is_initialized():
            dist.barrier(group=self.group)
        for full, _dsts, own, peers in self._peer.values():
            for pp in peers:
                _lib.call("tw_ipc_close", pp)
            _lib.call("tw_ipc_free", own)
        self._peer.clear()

    def _stream_barrier(self, stream):
        """All ranks reach this point of their streams before any continues.
        NCCL: a one-element all-reduce queued on the stream -- a device-side
        barrier, no host round trip.  gloo (several ranks sharing a device in
        the CPU/1-GPU tests): host barrier after draining the device."""
        if dist.get_backend(self.group) == "nccl":
            flag = self.__dict__.get("_flag")
            if flag is None:
                flag = self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
            ctx = torch.cuda.stream(stream) if isinstance(stream, torch.cuda.Stream) else contextlib.nullcontext()
            with ctx:
                dist.all_reduce(flag, group=self.group)
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)

    def _gemm_fused(self, at, out_dtype, stream):
        m = at.shape[1]
        full, dsts, _own, _peers = self._peer_buffers(m, out_dtype)
        width = self.col_range[1] - self.col_range[0]
        # peers are done reading the previous result from their replicas
        self._stream_barrier(stream)
        if width and m:
            if at.dtype != self.plan.dtype or at.dim() != 2 or at.shape[0] != self.k:
                raise DimensionError(f"A^T must be a ({self.k}, M) {self.plan.dtype} CUDA tensor")
            _lib.call("tw_gemm_peers", self.plan._h, at.data_ptr(), m, at.stride(0), ctypes.cast(dsts, ctypes.c_void_p),
                      self.world, m,
                      _code(out_dtype), _stream_ptr(stream, self.device))
        # every rank's kernel (queued before the barrier on its stream) has
        # finished storing into every replica
        self._stream_barrier(stream)
        return full[: self.n]

    def gemm(self, at, out_dtype=None, stream=None):
        """Full C^T (N x M) on every rank: per round, TW-GEMM into this
        rank's slot, then an in-place all-gather of the round's rows.
        `stream`: a torch.cuda.Stream (or None for the current stream)."""
        out_dtype = out_dtype or torch.float32
        if self.fused and self.world > 1:
            return self._gemm_fused(at, out_dtype, stream)
        full = self._full(at.shape[1], out_dtype)
        rows = self.world * self.chunk
        pending = []
        # NCCL orders each collective after the work queued on the current
        # stream, so the GEMMs run on it too
        ctx = torch.cuda.stream(stream) if isinstance(stream, torch.cuda.Stream) else contextlib.nullcontext()
        with ctx:
            for j in range(self.rounds):
                self._compute(at, full, j, out_dtype, None)
                if self.world > 1:
                    pending.append(_gather_round(full[j * rows:(j + 1) * rows], self._slot(full, j), self.group))
            for wk in pending:
                if wk is not None:
                    wk.wait()
        return full[: self.n]


class _CudaArray:
    """__cuda_array_interface__ wrapper: a torch view of a raw device buffer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _device_view(ptr, shape, dtype, device):
    typestr = {torch.float32: "<f4", torch.float16: "<f2", torch.bfloat16: "<f2"}[dtype]
    t = torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


def _gather_round(dst, mine, group):
    """All-gather equal row blocks into `dst`, `mine` being this rank's block
    inside it (in place).  NCCL: asynchronous, ordered after the GEMM on the
    current stream.  gloo (host-logic tests): staged through the host."""
    if mine.is_cuda and dist.get_backend(group) == "nccl":
        return dist.all_gather_into_tensor(dst, mine, group=group, async_op=True)
    host = torch.empty(dst.shape, dtype=dst.dtype)
    dist.all_gather_into_tensor(host, mine.contiguous().cpu(), group=group)
    dst.copy_(host)
    return None


def shard_table(n: int, world: int) -> np.ndarray:
    """(world, 2) int64 array of the shard ranges (for logs and tests)."""
    return np.asarray(shard_ranges(n, world), np.int64).reshape(world, 2)
