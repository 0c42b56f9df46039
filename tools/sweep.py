"""Throughput sweep over every BASELINE.json config (B200, 1 GPU).

    python tools/sweep.py [--quick] [--out profiles/r01_sweep]

Rows:
  C1   M=N=K=1024, G=128, 50% TW (the reference's CPU-runnable oracle case)
  C2a  BERT-base FC1 4096x768x3072 @75%     C2b  BERT-base 4096x768x768 @75%
  C3   VGG-16 conv layers as im2col GEMMs, batch 64 (M = 64*H*W, K = 9*Cin,
       N = Cout) at 50% and 75% TW
  C4   TEW on BERT-base FC1: 76.5% TW + 1.5% element-wise overlay (CSC)
  C5   BERT-large FC1 16384x1024x4096, sparsity 0 / .1 / .25 / .5 / .75 / .9
  NMT  LSTM gate GEMM of a 512-unit layer, [x;h] (K=1024) -> 4 gates (N=2048),
       4096 tokens, at 50 / 75 / 90% -- an assumed shape (PAPER.md:626-627
       gives none)

Per row: TW kernel time (CUDA events, mean of `reps` launches over rotating
output buffers when the output is smaller than 2x L2; calls graph-captured and replayed), fp32 and fp16 output;
dense cuBLAS bf16 (torch.mm, bf16 out) at the same shape; dense-equivalent
and kept TFLOPS; algorithmic HBM bytes and GB/s; speedup vs cuBLAS.  Parity:
rel-L2 of the fp32 output against the CPU oracle on a token slice (the first
min(M, 1024) tokens), pruned columns exactly zero.  Synthetic data: A, W ~
N(0,1) rounded to bf16; patterns from the reference's random_uniform_pattern
(seed 42).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_13006_b200 as tw  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (checker only)

L2 = 126 * 2**20
VGG = [  # (name, H, Cin, Cout)
    ("conv1_1", 224, 3, 64), ("conv1_2", 224, 64, 64), ("conv2_1", 112, 64, 128), ("conv2_2", 112, 128, 128),
    ("conv3_1", 56, 128, 256), ("conv3_2", 56, 256, 256), ("conv3_3", 56, 256, 256), ("conv4_1", 28, 256, 512),
    ("conv4_2", 28, 512, 512), ("conv4_3", 28, 512, 512), ("conv5_1", 14, 512, 512), ("conv5_2", 14, 512, 512),
    ("conv5_3", 14, 512, 512),
]


def rows(quick: bool):
    r = [("C1", 1024, 1024, 1024, 0.50, None), ("C2a", 4096, 768, 3072, 0.75, None),
         ("C2b", 4096, 768, 768, 0.75, None), ("C4-TEW", 4096, 768, 3072, 0.765, 0.015),
         ("C2a-het", 4096, 768, 3072, 0.75, None), ("C5-het@0.75", 16384, 1024, 4096, 0.75, None)]
    for s in (0.5, 0.75, 0.9):
        r.append((f"NMT@{s:g}", 4096, 1024, 2048, s, None))
    for s in ([0.0, 0.25, 0.4, 0.5, 0.75, 0.9] if quick else [0.0, 0.1, 0.25, 0.4, 0.5, 0.75, 0.9]):
        r.append((f"C5@{s:g}", 16384, 1024, 4096, s, None))
    vgg = VGG[1::3] if quick else VGG
    for s in (0.5, 0.75):
        for name, hw, cin, cout in vgg:
            r.append((f"C3 {name}@{s:g}", 64 * hw * hw, 9 * cin, cout, s, None))
    return r


def timed(fn, reps):
    """us per call: `reps` calls captured into one CUDA graph and replayed
    (kernel time without per-call host launch overhead, as in bench.py)."""
    for i in range(2):
        fn(i)
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
    return a.elapsed_time(b) / reps * 1e3  # us


def run_row(name, m, k, n, s, delta, reps, hbm_peak):
    g = 128
    rng = np.random.default_rng(42)
    w = orc.bf16_round(rng.standard_normal((k, n)).astype(np.float32))
    p = orc.random_uniform_pattern(k, n, g, s, 42)
    if "-het" in name:
        # non-uniform tiles: each tile keeps k_i = kbar * U(0.85, 1.15)
        # rows, so units differ in cost and the LPT schedule has to balance them
        hr = np.random.default_rng(7)
        tiles = []
        for cols, keep in p[3]:
            kk = int(np.clip(round(keep.sum() * hr.uniform(0.85, 1.15)), 1, k))
            nk = np.zeros(k, bool)
            nk[np.sort(hr.choice(k, size=kk, replace=False))] = True
            tiles.append((cols, nk))
        p = (p[0], p[1], p[2], tiles)
    ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
    plan = tw.TwPlan(ts)
    info = plan.info
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(42)
    ld = (m + 7) // 8 * 8
    at = torch.randn((k, ld), generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)[:, :m]
    csc = None
    if delta:
        cp, ri, va = orc.tew_overlay_magnitude(w, p, delta)
        csc = tw.DeviceCsc(tw.CscMatrix(k, n, cp, ri, va))
    out_bytes32 = 4 * m * n
    n_sets = 1 if out_bytes32 > 2 * L2 else int(np.ceil(2 * L2 / out_bytes32)) + 1
    res = {"row": name, "m": m, "k": k, "n": n, "sparsity": s, "live_tiles": info["n_live"],
           "element_sparsity": 1 - info["kept_elems"] / (k * n)}
    for od, dt in (("fp32", torch.float32), ("fp16", torch.float16)):
        outs = [torch.empty((n, m), dtype=dt, device=dev) for _ in range(n_sets)]
        if csc is None:
            us = timed(lambda i: plan.gemm(at, out=outs[i % n_sets], out_dtype=dt), reps)
        else:
            us = timed(lambda i: plan.gemm_tew(at, csc, out=outs[i % n_sets], out_dtype=dt), reps)
        q = bench.algorithmic_bytes(info, m, 4 if od == "fp32" else 2) + (
            (6 * csc.nnz + 4 * (n + 1)) if csc is not None else 0)
        res[f"us_{od}"] = us
        res[f"gbs_{od}"] = q / (us * 1e-6) / 1e9
        res[f"hbm_frac_{od}"] = res[f"gbs_{od}"] / hbm_peak
        if od == "fp32":
            ct_slice = outs[0][:, : min(m, 1024)].float().cpu().numpy()
        del outs
    # which kernel the (auto) plan runs at this M: 2 = K2 gathers, 4 = K4 CTA pairs
    if csc is None:
        res["kernel"] = plan._for_launch(m, torch.float16).kernel_for(m, torch.float16)
    else:
        mp = plan.__dict__.get("_tew_plans", {}).get(csc)
        res["kernel"] = mp._for_launch(m, torch.float16).kernel_for(m, torch.float16) if mp is not None else 2
    # parity on a token slice
    ms = min(m, 1024)
    at32 = at[:, :ms].float().cpu().numpy()
    want = orc.gemm_tw_ct(np.ascontiguousarray(at32), orc.PackedTiles(orc.compact(w, p), k, n),
                          threads=orc.max_threads())
    if csc is not None:
        want = orc.gemm_tew_ct(np.ascontiguousarray(at32), orc.PackedTiles(orc.compact(w, p), k, n),
                               *orc.tew_overlay_magnitude(w, p, delta), threads=orc.max_threads())
    res["rel_l2"] = orc.rel_l2(ct_slice, want)
    pr = orc.pruned_columns(p)
    res["pruned_zero"] = bool(np.all(ct_slice[pr] == 0.0)) if csc is None else None
    # dense cuBLAS bf16 at the same shape
    a_rm = at.t().contiguous() if m * k * 2 < 8 * 2**30 else None
    wd = torch.from_numpy(w).to(dev, torch.bfloat16)
    if a_rm is not None:
        cd = [torch.empty((m, n), dtype=torch.bfloat16, device=dev) for _ in range(max(1, n_sets))]
        res["us_cublas_bf16"] = timed(lambda i: torch.mm(a_rm, wd, out=cd[i % len(cd)]), reps)
        del cd, a_rm
    flops_d = 2 * m * k * n
    flops_k = 2 * m * info["kept_elems"] + (2 * m * csc.nnz if csc is not None else 0)
    res["tflops_dense_fp32"] = flops_d / (res["us_fp32"] * 1e-6) / 1e12
    res["tflops_kept_fp32"] = flops_k / (res["us_fp32"] * 1e-6) / 1e12
    if "us_cublas_bf16" in res:
        res["speedup_fp16_vs_cublas_bf16"] = res["us_cublas_bf16"] / res["us_fp16"]
        res["speedup_fp32_vs_cublas_bf16"] = res["us_cublas_bf16"] / res["us_fp32"]
    del at
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep"))
    ap.add_argument("--only", default=None, help="substring filter on row names")
    args = ap.parse_args()
    hbm_peak, _, _ = bench.load_peaks()
    results = []
    for r in rows(args.quick):
        if args.only and args.only not in r[0]:
            continue
        t0 = time.time()
        res = run_row(*r, reps=args.reps, hbm_peak=hbm_peak)
        res["wall_s"] = time.time() - t0
        results.append(res)
        print(json.dumps(res), flush=True)
    with open(args.out + ".json", "w") as f:
        json.dump(results, f, indent=1)
    lines = ["| row | M | K | N | elem. sparsity | kernel | TW fp32 µs | TW fp16 µs | cuBLAS bf16 µs | fp16 speedup | "
             "fp32 GB/s (frac) | dense-eq TFLOPS (fp32) | rel-L2 |", "|" + "---|" * 13]
    for r in results:
        cub = r.get("us_cublas_bf16")
        lines.append(
            f"| {r['row']} | {r['m']} | {r['k']} | {r['n']} | {r['element_sparsity']:.3f} | K{r['kernel']} | {r['us_fp32']:.1f} | "
            f"{r['us_fp16']:.1f} | {cub:.1f} | {r['speedup_fp16_vs_cublas_bf16']:.2f}x | "
            f"{r['gbs_fp32']:.0f} ({r['hbm_frac_fp32']:.2f}) | {r['tflops_dense_fp32']:.0f} | {r['rel_l2']:.1e} |"
            if cub else
            f"| {r['row']} | {r['m']} | {r['k']} | {r['n']} | {r['element_sparsity']:.3f} | K{r['kernel']} | {r['us_fp32']:.1f} | "
            f"{r['us_fp16']:.1f} | — | — | {r['gbs_fp32']:.0f} ({r['hbm_frac_fp32']:.2f}) | "
            f"{r['tflops_dense_fp32']:.0f} | {r['rel_l2']:.1e} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
