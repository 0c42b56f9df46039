"""K2 (kept-row gathers) vs K4 (dense-padded CTA pairs) vs cuBLAS bf16 across
sparsity, timed in interleaved rounds so all three arms see the same clocks
(the tensor-heavy near-dense runs hit the board power cap).  Sets the
TwPlan(dense_pad=None) threshold (engine.DENSE_PAD_MIN_DENSITY).

    python tools/pad_sweep.py [--shape C5|C2a] [--rounds 5]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_13006_b200 as tw  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (inputs + parity slice only)

SHAPES = {"C5": (16384, 1024, 4096), "C2a": (4096, 768, 3072), "NMT": (4096, 1024, 2048)}


def graph_us(fn, reps):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="C5", choices=sorted(SHAPES))
    ap.add_argument("--sparsity", default="0,0.1,0.2,0.3,0.4,0.5,0.6")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tew", action="store_true", help="C4: TEW merged plans (76.5%% TW + 1.5%% overlay)")
    args = ap.parse_args()
    m, k, n = SHAPES[args.shape]
    dev = torch.device("cuda")
    L2 = 126 * 2**20
    n_sets = max(2, int(np.ceil(2 * L2 / (2 * m * n + 2 * m * k))) + 1)
    gen = torch.Generator(device=dev).manual_seed(1)
    ats = [torch.randn((k, m), generator=gen, device=dev).to(torch.bfloat16) for _ in range(n_sets)]
    outs = [torch.empty((n, m), dtype=torch.float16, device=dev) for _ in range(n_sets)]
    a_rm = [x.t().contiguous() for x in ats]
    cub_out = [torch.empty((m, n), dtype=torch.bfloat16, device=dev) for _ in range(n_sets)]
    sps = [0.765] if args.tew else [float(x) for x in args.sparsity.split(",")]
    for s in sps:
        rng = np.random.default_rng(42)
        w = orc.bf16_round(rng.standard_normal((k, n)).astype(np.float32))
        p = orc.random_uniform_pattern(k, n, 128, s, 42)
        ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
        wd = torch.from_numpy(w).to(dev, torch.bfloat16)
        arms = {}
        if args.tew:  # the merged plan gemm_tew runs (tw + overlay as one tile set)
            ts = tw.engine.tew_merged_tileset(ts, tw.CscMatrix(k, n, *orc.tew_overlay_magnitude(w, p, 0.015)))
        for name, pad in (("K2", False), ("K4", True)):
            plan = tw.TwPlan(ts, dense_pad=pad)
            arms[name] = (lambda pl: lambda i: pl.gemm(ats[i % n_sets], out=outs[i % n_sets],
                                                       out_dtype=torch.float16))(plan)
        arms["cublas"] = lambda i: torch.mm(a_rm[i % n_sets], wd, out=cub_out[i % n_sets])
        t = {x: [] for x in arms}
        for _ in range(args.rounds):
            for x, fn in arms.items():
                t[x].append(graph_us(fn, args.reps))
        med = {x: statistics.median(v) for x, v in t.items()}
        info = tw.TwPlan(ts, dense_pad=False).info
        dens = info["kept_elems"] / (k * max(1, info["sum_n"]))
        print(json.dumps({"shape": args.shape, "sparsity": s, "tile_density": round(dens, 3),
                          **{f"us_{x}": round(v, 2) for x, v in med.items()},
                          "K4_vs_K2": round(med["K2"] / med["K4"], 3),
                          "best_vs_cublas": round(med["cublas"] / min(med["K2"], med["K4"]), 3)}), flush=True)


if __name__ == "__main__":
    main()
