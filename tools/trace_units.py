"""Per-CTA / per-unit timeline of one tw_gemm launch (tw_gemm_traced hook).

    python tools/trace_units.py --workload C2a [--out-dtype fp32]

Prints, relative to the earliest stamp in the launch: when each role starts
and finishes its units, so stalls can be attributed to the producer (gather),
the MMA issuer or the epilogue (stores / zero rows).
"""

from __future__ import annotations

import argparse
import ctypes
import json
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

SLOTS = ["prod_start", "prod_issued", "mma_start", "mma_commit", "epi_zero_done", "epi_acc_ready", "epi_stored"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2a")
    ap.add_argument("--out-dtype", default="fp32")
    ap.add_argument("--json", default=None)
    ap.add_argument("--pad", type=int, default=0, help="extra elements per A^T row (row pitch)")
    ap.add_argument("--cold", action="store_true", help="evict the output from L2 before the traced launch")
    ap.add_argument("--m", type=int, default=0, help="override the token count M")
    ap.add_argument("--soak", action="store_true", help="traced launch queued behind ~0.3 s of launches (full clocks)")
    args = ap.parse_args()
    m, k, n, g, s, _ = bench.WORKLOADS[args.workload]
    m = args.m or m
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
    ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
    plan = tw.TwPlan(ts)
    if args.pad:
        buf = torch.empty((k, m + args.pad), dtype=torch.bfloat16, device="cuda")[:, :m]
        at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16, out=buf)
    else:
        at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    dt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[args.out_dtype]
    out = torch.empty((n, m), dtype=dt, device="cuda")
    sms_dev = ctypes.c_int(0)
    _lib.call("tw_device_sm_count", ctypes.byref(sms_dev))
    # the trace is indexed by the launch grid (the schedule's CTA count)
    _, unit_off, _ = plan.schedule(m, args.out_dtype, sms=int(os.environ.get("TW_B200_SMS", sms_dev.value)))
    sms = ctypes.c_int(len(unit_off) - 1)
    trace = torch.zeros(sms.value * (64 + 128 + 32), dtype=torch.int64, device="cuda")
    code = {"fp32": 0, "bf16": 1, "fp16": 2}[args.out_dtype]
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        plan.gemm(at, out=out, out_dtype=dt)
    torch.cuda.synchronize()
    # clock soak: ~0.3 s of back-to-back launches, the traced one queued right behind
    soak = [torch.empty_like(out) for _ in range(4)]
    for i in range(20000 if args.soak else 0):
        plan.gemm(at, out=soak[i % 4], out_dtype=dt)
    others = [torch.empty_like(out) for _ in range(5)] if args.cold else []
    ats = [at.clone() for _ in range(5)] if args.cold else []
    if not args.soak:
        torch.cuda.synchronize()
    trace.zero_()
    # --cold: back-to-back launches on rotating buffers right before the traced
    # one, with no sync in between (bench.py's steady state)
    for o, a2 in zip(others, ats):
        plan.gemm(a2, out=o, out_dtype=dt)
    _lib.call("tw_gemm_traced", plan._h, at.data_ptr(), m, at.stride(0), out.data_ptr(), out.stride(0), code,
              trace.data_ptr(), stream)
    torch.cuda.synchronize()
    full = trace.cpu().numpy().astype(np.float64)
    tr = full[: sms.value * 64].reshape(sms.value, 8, 8)
    st = full[sms.value * 64: sms.value * 192].reshape(sms.value, 32, 4)
    ep = full[sms.value * 192:].reshape(sms.value, 32)
    tr = tr.copy()
    tr[:, 7, 2:4] = 0  # clock64 samples, not timestamps
    valid = tr > 0
    t0 = tr[valid].min()
    rel = np.where(valid, (tr - t0) / 1e3, np.nan)  # us
    print(f"launch span {np.nanmax(rel):.2f} us over {sms.value} CTAs")
    summary = {}
    for si, name in enumerate(SLOTS):
        for ui in range(4):
            col = rel[:, ui, si]
            if np.isfinite(col).any():
                summary[f"u{ui}.{name}"] = [float(np.nanmin(col)), float(np.nanmedian(col)), float(np.nanmax(col))]
    for kk, v in summary.items():
        print(f"{kk:22s} min {v[0]:8.2f}  med {v[1]:8.2f}  max {v[2]:8.2f}")
    srel = np.where(st > 0, (st - t0) / 1e3, np.nan)
    print("stage  issued(med)  full(med)  committed(med)   [CTA 0: issued full committed]")
    for si in range(14):
        c0 = srel[0, si]
        print(f"{si:5d} {np.nanmedian(srel[:, si, 0]):9.2f} {np.nanmedian(srel[:, si, 1]):9.2f} "
              f"{np.nanmedian(srel[:, si, 2]):9.2f}     [{c0[0]:7.2f} {c0[1]:7.2f} {c0[2]:7.2f}]")
    raw3 = full[sms.value * 64: sms.value * 192].reshape(sms.value, 32, 4)[:, :, 3].astype(np.int64)
    print("producer cycles per stage (median over CTAs): wait_empty wait_idx index_lds issue")
    for si in range(12):
        v = raw3[:, si]
        v = v[v > 0]
        if v.size:
            print(f"  stage {si:2d}: {np.median(v >> 48):7.0f} {np.median((v >> 32) & 0xffff):7.0f} "
                  f"{np.median((v >> 16) & 0xffff):7.0f} {np.median(v & 0xffff):7.0f}")
    base = np.where(ep[:, 28:29] > 0, ep[:, 28:29], np.nan)  # bulk epilogue entry
    erel = np.where(ep > 0, ep - base, np.nan)  # SM cycles since chunk 0's TMEM load completed
    print("bulk epilogue of unit 0, pass c (median over CTAs, SM cycles from entry): staging free / staged / synced / issued")
    for c in range(2):
        row = [np.nanmedian(erel[:, c * 4 + x]) if np.isfinite(erel[:, c * 4 + x]).any() else float("nan") for x in range(4)]
        print(f"  chunk {c}: " + " ".join(f"{v:8.0f}" for v in row))
    # SM clock during the launch: clock64 vs globaltimer between CTA start and end
    ck = full[: sms.value * 64].reshape(sms.value, 8, 8)[:, 7, :4]
    ok = (ck[:, 0] > 0) & (ck[:, 1] > ck[:, 0]) & (ck[:, 3] > ck[:, 2])
    if ok.any():
        mhz = (ck[ok, 3] - ck[ok, 2]) / (ck[ok, 1] - ck[ok, 0]) * 1e3
        print(f"SM clock during the launch: median {np.median(mhz):.0f} MHz (min {mhz.min():.0f}, max {mhz.max():.0f})")
    ends = rel[:, 7, :3]
    print("CTA start / zeros issued / drained (min med max):",
          [(round(float(np.nanmin(ends[:, i])), 2), round(float(np.nanmedian(ends[:, i])), 2),
            round(float(np.nanmax(ends[:, i])), 2)) for i in range(3)])
    # per-unit durations
    mma = rel[:, :, 3] - rel[:, :, 2]
    prod = rel[:, :, 1] - rel[:, :, 0]
    store = rel[:, :, 6] - rel[:, :, 5]
    print(f"producer issue time/unit med {np.nanmedian(prod):.2f} us; MMA issue/unit med {np.nanmedian(mma):.2f}; "
          f"epilogue store/unit med {np.nanmedian(store):.2f}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"summary": summary, "raw_us": np.nan_to_num(rel, nan=-1).tolist()}, f)


if __name__ == "__main__":
    main()
