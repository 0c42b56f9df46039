"""Probe: pair neighbouring G=128 tiles into 256-column tiles over the UNION of
their kept rows (zero-padded weights), run by the BN=256 instantiation (two
M=128 MMAs share every gathered A^T stage; 128-token units).  Per output
element the gathered A^T bytes halve relative to the 128-column / 256-token
unit, the weight bytes double -- worth it when the gathers dominate and the
masks overlap (near-dense, moderate sparsity).

    python tools/pair_probe.py --workload C2a [--reps 50]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_13006_b200 as tw  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from tools.sweep import timed  # noqa: E402


def paired_tileset(ts):
    k, n = ts.k, ts.n
    out = []
    tiles = list(ts.tiles)
    for i in range(0, len(tiles), 2):
        grp = tiles[i:i + 2]
        keeps = [tw.unpack_mask_words(t.row_mask_words, k).astype(bool) for t in grp]
        keep = np.logical_or.reduce(keeps)
        rows = np.flatnonzero(keep)
        cols = np.concatenate([np.asarray(t.col_ids, np.int32) for t in grp])
        sub = np.zeros((rows.size, cols.size), np.float32)
        c0 = 0
        for t, kp in zip(grp, keeps):
            sm = np.asarray(t.sub_matrix.data, np.float32).reshape(t.sub_matrix.cols, t.sub_matrix.rows).T
            pos = np.searchsorted(rows, np.flatnonzero(kp))
            sub[pos, c0:c0 + sm.shape[1]] = sm
            c0 += sm.shape[1]
        out.append(tw.CompactTile(sub_matrix=tw.DenseMatrix(rows.size, cols.size, tw.Layout.COL_MAJOR,
                                                              np.ascontiguousarray(sub.T).reshape(-1)),
                                  row_mask_words=tw.pack_mask_words(keep), col_ids=cols))
    return tw.CompactTileSet(k, n, 256, tuple(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", nargs="+", default=["C2a"])
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    for wl in args.workload:
        m, k, n, g, s, _ = bench.WORKLOADS[wl]
        a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
        ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
        pts = paired_tileset(ts)
        at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
        n_sets = max(2, int(np.ceil(2 * bench.L2_BYTES / (2 * n * m))) + 1)
        outs = [torch.empty((n, m), dtype=torch.float16, device="cuda") for _ in range(n_sets)]
        res = {}
        ref = None
        for name, t in (("g128", ts), ("paired_g256", pts)):
            plan = tw.TwPlan(t)
            us = timed(lambda i: plan.gemm(at, out=outs[i % n_sets], out_dtype=torch.float16), args.reps)
            got = plan.gemm(at, out_dtype=torch.float32)[:, :512].cpu().numpy()
            if ref is None:
                ref = orc.gemm_tw_ct(np.ascontiguousarray(a[:512].T), orc.PackedTiles(orc.compact(w, p), k, n),
                                     threads=orc.max_threads())
            res[name] = (us, orc.rel_l2(got, ref), plan.info["sum_k"], plan.info["wimg_bytes"])
        print(wl, {kk: f"{v[0]:.2f} us rel {v[1]:.1e} sum_k {v[2]} wimg {v[3] / 2**20:.1f} MB" for kk, v in res.items()},
              flush=True)


if __name__ == "__main__":
    main()
