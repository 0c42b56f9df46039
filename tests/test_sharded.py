"""N-sharded multi-GPU path -- host logic on CPU.

world_size 2 and 3 `gloo` process groups (127.0.0.1): every rank packs its
column-range shard of the layer with the product packer, evaluates that
packed shard on the CPU (test-side emulation of the kernel from the packed
image: kept-K lists, column ids, swizzled weights, zero rows), and the
product's all_gather_rows reassembles C^T.  The result must equal the
oracle's full-layer gemm_tw within bf16-operand tolerance, with pruned
columns exactly zero -- i.e. the shards partition the layer and the gather
puts every row where the reference's COL_MAJOR C buffer has it."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2008_13006_b200 as tw
from paper_2008_13006_b200 import sharded
from oracle import oracle as orc
from tests.test_packer import decode_wimg, to_tw_pattern


def test_shard_ranges():
    assert sharded.shard_ranges(3072, 8) == [(384 * r, 384 * (r + 1)) for r in range(8)]
    assert sharded.shard_ranges(1000, 3) == [(0, 334), (334, 668), (668, 1000)]
    assert sharded.shard_ranges(5, 4) == [(0, 2), (2, 4), (4, 5), (5, 5)]
    assert sharded.shard_ranges(0, 2) == [(0, 0), (0, 0)]
    with pytest.raises(tw.DimensionError):
        sharded.shard_ranges(10, 0)


def emulate_shard(plan: tw.PackedPlan, at32: np.ndarray) -> np.ndarray:
    """C^T rows of one packed shard, computed from the packed image (float64)."""
    m = at32.shape[1]
    rows = plan.col_end - plan.col_begin
    ct = np.full((rows, m), np.nan, np.float64)
    table = plan.export("tiles")
    kidx, colids, zero, wimg = plan.export("kidx"), plan.export("colids"), plan.export("zero_rows"), plan.export("wimg")
    ct[zero] = 0.0
    if len(table):
        wrows = (wimg.size // int(table[:, 6].sum())) // 128
    for _src, koff, coff, n_i, k_i, _k16, nkb, woff in table:
        dec = decode_wimg(wimg[woff: woff + nkb * wrows * 128], wrows, nkb, n_i, k_i)
        w = (dec[:k_i, :n_i].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        ct[colids[coff: coff + n_i]] = w.T @ at32[kidx[koff: koff + k_i]].astype(np.float64)
    assert not np.isnan(ct).any(), "shard leaves output rows unwritten"
    return ct.astype(np.float32)


def _worker(rank, world, port, m, k, n, s, seed, q, rounds=1):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        a, w, p = orc.bench_inputs(m, k, n, 128, s, seed=seed)
        ts = tw.compact(tw.DenseMatrix.from_array(w), to_tw_pattern(p))
        at32 = np.ascontiguousarray(a.T)
        kept = torch.zeros(1, dtype=torch.int64)
        if rounds == 1:
            c0, c1 = sharded.shard_ranges(n, world)[rank]
            plan = tw.PackedPlan(ts, col_range=(c0, c1))
            per = sharded.rows_per_rank(n, world)
            local = torch.zeros((per, m), dtype=torch.float32)
            local[: c1 - c0] = torch.from_numpy(emulate_shard(plan, at32))
            full = sharded.all_gather_rows(local, n)
            kept += plan.info["kept_elems"]
        else:
            # block-cyclic rounds, gathered in place round by round
            chunks = sharded.cyclic_ranges(n, world, rounds)
            sz = -(-n // (world * rounds))
            buf = torch.zeros((sz * world * rounds, m), dtype=torch.float32)
            for j, (c0, c1) in enumerate(chunks[rank]):
                c = j * world + rank
                assert c0 == min(n, c * sz)
                if c1 > c0:
                    plan = tw.PackedPlan(ts, col_range=(c0, c1))
                    buf[c * sz: c * sz + c1 - c0] = torch.from_numpy(emulate_shard(plan, at32))
                    kept += plan.info["kept_elems"]
                sharded._gather_round(buf[j * world * sz:(j + 1) * world * sz], buf[c * sz:(c + 1) * sz], None)
            full = buf[:n]
        assert full.shape == (n, m) and full.is_contiguous()
        dist.all_reduce(kept)
        if rank == 0:
            want = orc.gemm_tw_ct(np.ascontiguousarray(a.T), orc.PackedTiles(orc.compact(w, p), k, n))
            got = full.numpy()
            q.put(("ok", orc.rel_l2(got, want), bool(np.all(got[orc.pruned_columns(p)] == 0.0)),
                   int(kept.item()), int(sum(ci.size * np.count_nonzero(kp) for ci, kp in p[3]))))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e)))
        raise


def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_cyclic_ranges():
    # 2 ranks x 3 rounds over 1000 columns: chunk 167, rank r owns chunks r, 2+r, 4+r
    cr = sharded.cyclic_ranges(1000, 2, 3)
    assert cr[0] == [(0, 167), (334, 501), (668, 835)]
    assert cr[1] == [(167, 334), (501, 668), (835, 1000)]
    assert sharded.cyclic_ranges(3072, 8, 1) == [[r] for r in sharded.shard_ranges(3072, 8)]
    # every column owned exactly once
    for n, w, j in [(1000, 3, 4), (7, 4, 3), (4096, 8, 4), (0, 2, 2)]:
        cols = sorted(c for rk in sharded.cyclic_ranges(n, w, j) for a, b in rk for c in range(a, b))
        assert cols == list(range(n))
    with pytest.raises(tw.DimensionError):
        sharded.cyclic_ranges(10, 2, 0)


@pytest.mark.parametrize("world,m,k,n,s,rounds", [(2, 96, 256, 1000, 0.75, 1), (3, 64, 200, 700, 0.5, 1),
                                                  (2, 64, 256, 1000, 0.75, 3)])
def test_gloo_sharded_layer_reassembles(world, m, k, n, s, rounds):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, k, n, s, 7, q, rounds)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
    assert res[0] == "ok", res
    _, err, zeros_ok, kept, kept_want = res
    assert err < 1e-5  # same bf16-rounded operands; only the accumulation order differs
    assert zeros_ok
    assert kept == kept_want
    assert all(pr.exitcode == 0 for pr in procs)


def test_fused_mode_needs_contiguous_ranges():
    # the peer-store (fused all-gather) path writes each rank's contiguous
    # column range into every replica; block-cyclic rounds are rejected
    a, w, p = orc.bench_inputs(16, 64, 256, 128, 0.5, seed=3)
    ts = tw.compact(tw.DenseMatrix.from_array(w), to_tw_pattern(p))
    with pytest.raises(tw.DimensionError):
        sharded.ShardedTwPlan(ts, rounds=2, fused=True)
