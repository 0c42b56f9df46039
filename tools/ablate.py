"""Ablation timings of the TW kernel at full clocks: the same rotating-buffer,
graph-replayed timing as bench.py, through the tw_gemm_traced entry point
(the only one that honours the TW_B200_DEBUG experiment bits:
1 skip zero rows, 2 skip kept-row stores, 4 skip MMA, 64 skip weight copies,
256 force the zero-fill gather path).  Results are NOT parity-valid; they
attribute the step time to gathers / MMA / stores.

    python tools/ablate.py --workload C2a --out-dtype fp16 --debug 0 1 2 3 4 64
"""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_13006_b200 as tw  # noqa: E402
from paper_2008_13006_b200 import _lib  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2a")
    ap.add_argument("--out-dtype", default="fp16")
    ap.add_argument("--debug", type=int, nargs="+", default=[0, 1, 2, 3, 4, 64])
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warm-a", action="store_true", help="one A^T for every step (L2-resident input)")
    ap.add_argument("--m", type=int, default=0, help="override the token count M")
    ap.add_argument("--hot", action="store_true", help="one plan / A^T / output for every step (all L2-resident)")
    args = ap.parse_args()
    m, k, n, g, s, _ = bench.WORKLOADS[args.workload]
    m = args.m or m
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
    ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
    dt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[args.out_dtype]
    code = {"fp32": 0, "bf16": 1, "fp16": 2}[args.out_dtype]
    ob = 4 if args.out_dtype == "fp32" else 2
    at0 = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    set_bytes = 2 * k * m + ob * n * m
    n_sets = max(2, int(np.ceil(2 * bench.L2_BYTES / set_bytes)) + 1)
    if args.hot:
        n_sets = 1
    plans = [tw.TwPlan(ts) for _ in range(n_sets)]
    ats = [at0] * n_sets if args.warm_a else [at0] + [at0.clone() for _ in range(n_sets - 1)]
    outs = [torch.empty((n, m), dtype=dt, device="cuda") for _ in range(n_sets)]
    trace = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")  # scratch (stamps are discarded)

    def step(i):
        j = i % n_sets
        st = torch.cuda.current_stream().cuda_stream
        _lib.call("tw_gemm_traced", plans[j]._h, ats[j].data_ptr(), m, ats[j].stride(0), outs[j].data_ptr(),
                  outs[j].stride(0), code, trace.data_ptr(), st)

    plain = bench.time_device(torch, lambda i: plans[i % n_sets].gemm(ats[i % n_sets], out=outs[i % n_sets],
                                                                     out_dtype=dt), args.steps, n_sets, soak_s=0.5)
    print(f"{args.workload} M={m} {args.out_dtype} plain tw_gemm{' (warm A)' if args.warm_a else ''}{' (hot)' if args.hot else ''}: {plain * 1e3:.2f} us")
    for d in args.debug:
        os.environ["TW_B200_DEBUG"] = str(d)
        ms = bench.time_device(torch, step, args.steps, n_sets, soak_s=0.3)
        print(f"{args.workload} M={m} {args.out_dtype} debug={d:4d}: {ms * 1e3:.2f} us")
    os.environ.pop("TW_B200_DEBUG", None)


if __name__ == "__main__":
    main()
