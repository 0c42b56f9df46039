"""Minimal launch sequence for ncu: the bench workload's TW-GEMM (and, with
--dense, the cuBLAS bf16 GEMM of the same shape) a few times, eagerly.

    ncu --set full --clock-control none --import-source on -k regex:tw_gemm \
        -s 3 -c 1 -o gpurun_out/prof python tools/ncu_step.py --workload C2a
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_13006_b200 as tw  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2a")
    ap.add_argument("--out-dtype", default="fp32")
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--tew", action="store_true")
    args = ap.parse_args()
    m, k, n, g, s, _ = bench.WORKLOADS[args.workload]
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
    ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
    plan = tw.TwPlan(ts)
    at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    dt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[args.out_dtype]
    out = torch.empty((n, m), dtype=dt, device="cuda")
    csc = None
    if args.tew:
        cp, ri, va = orc.tew_overlay_magnitude(w, p, 0.015)
        csc = tw.DeviceCsc(tw.CscMatrix(k, n, cp, ri, va))
    for _ in range(args.launches):
        if csc is not None:
            plan.gemm_tew(at, csc, out=out, out_dtype=dt)
        else:
            plan.gemm(at, out=out, out_dtype=dt)
    if args.dense:
        a_bf = torch.from_numpy(a).cuda().to(torch.bfloat16)
        w_bf = torch.from_numpy(w).cuda().to(torch.bfloat16)
        for _ in range(args.launches):
            torch.mm(a_bf, w_bf)
    torch.cuda.synchronize()
    print("done", plan.info)


if __name__ == "__main__":
    main()
