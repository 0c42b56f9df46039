"""GPU `verify` / `bench` commands with the reference CLI's flags, defaults,
CSV schema and exit codes (cli.py:46-59, :201-252, :348-425) -- SURVEY.md
§8(f) row 3.

    python -m paper_2008_13006_b200.cli verify --model m.twml --patterns DIR
    python -m paper_2008_13006_b200.cli bench --shapes 256,768,3072 --out b.csv

verify: `probes` random 32 x K probes per layer through the GPU TW-GEMM, each
compared with a float64 dense product of the same bf16-rounded operands
(north_star: outputs checked on identically rounded inputs); fails (exit 1)
when max|diff| > 1e-4 * K, the reference's tolerance (cli.py:372-377).
bench: per (shape, G, sparsity), the reference's BENCH_HEADER columns measured
on the GPU (dense = cuBLAS bf16 torch.mm, tw = this library; CUDA events,
median/mean/std of `repeats` after one warm-up, like engine.time_median),
plus GPU columns.  Exit codes: 0 ok, 1 verify failure, 2 config/dimension
error, 3 format / I/O error.
"""

from __future__ import annotations

import argparse
import csv
import os
import sys

import numpy as np

EXIT_OK, EXIT_VERIFY, EXIT_CONFIG, EXIT_IO = 0, 1, 2, 3
BENCH_HEADER = [
    "m", "k", "n", "g", "sparsity", "workers", "repeats",
    "dense_ms_median", "dense_ms_mean", "dense_ms_std",
    "tw_ms_median", "tw_ms_mean", "tw_ms_std",
    "flops", "dense_flops", "speedup", "max_abs_diff",
]
GPU_COLUMNS = ["device", "out_dtype", "tw_tflops_dense_equiv", "tw_tflops_kept", "algorithmic_gb_per_s"]


def _floats_csv(s):
    return tuple(float(x) for x in s.split(",") if x.strip())


def _ints_csv(s):
    return tuple(int(x) for x in s.split(",") if x.strip())


def _shapes(s):
    out = []
    for part in s.split(";"):
        dims = _ints_csv(part)
        if len(dims) != 3:
            raise ValueError(f"shape needs m,k,n, got {part!r}")
        out.append(dims)
    return tuple(out)


def _parser():
    p = argparse.ArgumentParser(prog="paper_2008_13006_b200.cli", description="B200 TW-GEMM verify / bench")
    sub = p.add_subparsers(dest="command", required=True)
    v = sub.add_parser("verify", help="random-probe oracle equivalence sweep (GPU)")
    v.add_argument("--model", required=True, help="TWML checkpoint")
    v.add_argument("--patterns", required=True, help="directory holding pattern_<i>.twpt files")
    v.add_argument("--probes", type=int, default=20)
    v.add_argument("--seed", type=int, default=42)
    v.add_argument("--workers", type=int, default=1)
    b = sub.add_parser("bench", help="dense (cuBLAS) vs tile-sparse (TW) timing sweep (GPU)")
    b.add_argument("--shapes", type=_shapes, default=((256, 768, 3072),))
    b.add_argument("--sparsities", type=_floats_csv, default=(0.0, 0.25, 0.5, 0.75, 0.9))
    b.add_argument("-g", "--granularity", type=_ints_csv, default=(128,))
    b.add_argument("--workers", type=int, default=1)
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--out", required=True, help="CSV output path")
    b.add_argument("--out-dtype", default="fp32", choices=["fp32", "fp16", "bf16"])
    return p


def _bf16(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).float().numpy()


def cmd_verify(ns) -> int:
    import torch

    from . import engine, formats
    from .matrix import DenseMatrix, DimensionError
    from .pattern import compact, zero_fill

    weights, _ = formats.read_model(ns.model)
    patterns = []
    for i in range(len(weights)):
        path = os.path.join(ns.patterns, f"pattern_{i}.twpt")
        if not os.path.exists(path):
            raise FileNotFoundError(f"missing pattern file {path}")
        patterns.append(formats.read_pattern(path))
    rng = np.random.default_rng(ns.seed)
    worst, m = 0.0, 32
    for w, p in zip(weights, patterns):
        if (p.k, p.n) != w.shape:
            raise DimensionError(f"pattern ({p.k},{p.n}) does not match weight {w.shape}")
        wr = _bf16(w)
        plan = engine.TwPlan(compact(DenseMatrix.from_array(wr), p))
        oracle_w = np.asarray(zero_fill(DenseMatrix.from_array(wr), p).array(), np.float64)
        tol = 1e-4 * p.k
        for _ in range(ns.probes):
            a = _bf16(rng.standard_normal((m, p.k)).astype(np.float32))
            at = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().to(torch.bfloat16)
            got = plan.gemm(at).t().cpu().numpy()
            want = a.astype(np.float64) @ oracle_w
            diff = float(np.max(np.abs(got - want))) if got.size else 0.0
            worst = max(worst, diff)
            if diff > tol:
                print(f"FAIL layer {p.k}x{p.n}: diff {diff:.3e} > tol {tol:.3e}")
                print(f"worst diff {worst:.3e}")
                return EXIT_VERIFY
    print(f"PASS {ns.probes} probes x {len(patterns)} layers, worst diff {worst:.3e}")
    return EXIT_OK


def _time(fn, repeats):
    import torch
    fn()  # warm-up (engine.time_median semantics)
    ts = []
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    arr = np.asarray(ts)
    return float(np.median(arr)), float(arr.mean()), float(arr.std())


def cmd_bench(ns) -> int:
    import torch

    from . import engine
    from .matrix import ConfigError, DenseMatrix
    from .pattern import compact, random_uniform_pattern, zero_fill

    if ns.repeats < 5:
        raise ConfigError(f"repeats must be >= 5, got {ns.repeats}")  # cli.py:383-384
    dt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[ns.out_dtype]
    rows = []
    for m, k, n in ns.shapes:
        for g in ns.granularity:
            for s in ns.sparsities:
                rng = np.random.default_rng(ns.seed)  # cli.py:408-411 input recipe
                a = _bf16(rng.standard_normal((m, k)).astype(np.float32))
                w = _bf16(rng.standard_normal((k, n)).astype(np.float32))
                p = random_uniform_pattern(k, n, g, s, ns.seed)
                ts = compact(DenseMatrix.from_array(w), p)
                plan = engine.TwPlan(ts)
                at = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().to(torch.bfloat16)
                out = torch.empty((n, m), dtype=dt, device="cuda")
                ad, wd = torch.from_numpy(a).cuda().to(torch.bfloat16), torch.from_numpy(w).cuda().to(torch.bfloat16)
                got = plan.gemm(at, out_dtype=torch.float32).t().cpu().numpy()
                want = a.astype(np.float64) @ np.asarray(zero_fill(DenseMatrix.from_array(w), p).array(), np.float64)
                diff = float(np.max(np.abs(got - want))) if got.size else 0.0
                dense = _time(lambda: torch.mm(ad, wd), ns.repeats)
                tw = _time(lambda: plan.gemm(at, out=out, out_dtype=dt), ns.repeats)
                flops = 2 * m * int(plan.info["kept_elems"])
                dflops = 2 * m * k * n
                qb = (2 * m * plan.info["union_k"] + 2 * plan.info["kept_elems"]
                      + (4 if ns.out_dtype == "fp32" else 2) * m * n)
                rows.append([m, k, n, g, s, ns.workers, ns.repeats, *(f"{x:.6f}" for x in dense),
                             *(f"{x:.6f}" for x in tw), flops, dflops, f"{dense[0] / tw[0]:.6f}", f"{diff:.6g}",
                             torch.cuda.get_device_name(), ns.out_dtype, f"{dflops / (tw[0] * 1e-3) / 1e12:.3f}",
                             f"{flops / (tw[0] * 1e-3) / 1e12:.3f}", f"{qb / (tw[0] * 1e-3) / 1e9:.1f}"])
                print(f"m={m} k={k} n={n} g={g} s={s} dense {dense[0]:.3f}ms tw {tw[0]:.3f}ms "
                      f"speedup {dense[0] / tw[0]:.3f} diff {diff:.3g}")
    with open(ns.out, "w", newline="") as f:
        wr = csv.writer(f)
        wr.writerow(BENCH_HEADER + GPU_COLUMNS)
        wr.writerows(rows)
    print(f"csv {ns.out}")
    return EXIT_OK


def main(argv=None) -> int:
    from .matrix import ConfigError, DimensionError, FormatError

    ns = _parser().parse_args(argv)
    try:
        return {"verify": cmd_verify, "bench": cmd_bench}[ns.command](ns)
    except (ConfigError, DimensionError) as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except FormatError as e:
        print(f"format error: {e}", file=sys.stderr)
        return EXIT_IO
    except OSError as e:
        print(f"io error: {e}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
