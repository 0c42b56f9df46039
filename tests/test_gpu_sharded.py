"""N-sharded layer on real kernels: two ranks (gloo process
group, both on cuda:0 -- the GPU box has one device) each run
ShardedTwPlan.gemm, i.e. the sm_100a kernel on a column-range plan, and
all_gather_rows reassembles C^T.  The result must equal the single-GPU
TwPlan output bit for bit (same kernel, same per-column arithmetic)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q, rounds, fused=False):
    try:
        import paper_2008_13006_b200 as tw
        from oracle import oracle as orc
        from tests.test_packer import to_tw_pattern

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        a, w, p = orc.bench_inputs(384, 512, 1000, 128, 0.75, seed=23)
        ts = tw.compact(tw.DenseMatrix.from_array(w), to_tw_pattern(p))
        at = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().to(torch.bfloat16)
        sp = tw.ShardedTwPlan(ts, rounds=rounds, fused=fused)
        full = sp.gemm(at, out_dtype=torch.float32)
        full = sp.gemm(at, out_dtype=torch.float32).clone()  # second call reuses the replicas
        torch.cuda.synchronize()
        if rank == 0:
            ref = tw.TwPlan(ts).gemm(at).cpu().numpy()
            q.put(("ok", bool(np.array_equal(full.cpu().numpy(), ref)), sp.chunks, tuple(full.shape)))
        dist.barrier()
        sp.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
        raise


@pytest.mark.parametrize("rounds,fused", [(1, False), (3, False), (1, True)])
def test_two_rank_sharded_gemm_on_gpu(rounds, fused):
    """fused=True: no collective -- each rank's kernel stores its rows into both
    ranks' C^T replicas through CUDA IPC peer pointers (tw_gemm_peers)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, rounds, fused)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
    assert res[0] == "ok", res
    assert res[1], "sharded output differs from the single-plan output"
    assert res[2] == ([(0, 500)] if rounds == 1 else [(0, 167), (334, 501), (668, 835)])
    assert res[3] == (1000, 384)
