"""Steady-state DRAM traffic per TW-GEMM launch, for bench.py's
`roofline.traffic` (SURVEY §8(d), B200_PROFILING.md "traffic").

Two modes:

  run   (under ncu) -- the bench's rotating-buffer steady state launched
        eagerly: n_sets input / output / plan sets whose total exceeds 2x L2,
        so every launch reads cold A^T and its output evicts earlier outputs.
            ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
                --cache-control none --clock-control none -k regex:tw_gemm -s 20 -c 40 \\
                --csv --log-file gpurun_out/traffic_C2a_fp16.csv \\
                python tools/ncu_traffic.py run --workload C2a --out-dtype fp16
        `--cache-control none` keeps L2 as the previous launch left it (no
        flush before a profiled kernel), and with three counters there is a
        single pass -- no replay -- so each launch sees exactly the cache
        state of the uninstrumented loop.
  merge -- reads those CSVs and writes profiles/ncu_traffic.json:
            {"C2a:fp16": {"bytes_per_launch": mean(read + write), "read": ...,
                          "write": ..., "launches": 40, "algorithmic": Q,
                          "ratio": traffic / Q, "source": <csv>}, ...}
        A DRAM write is counted when L2 evicts the line, i.e. often during a
        LATER launch; averaged over many launches of a steady rotation the
        per-launch mean is the launch's own write-back.
"""

from __future__ import annotations

import argparse
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(args):
    import numpy as np
    import torch

    import bench
    import paper_2008_13006_b200 as tw
    from oracle import oracle as orc

    m, k, n, g, s, _ = bench.WORKLOADS[args.workload]
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
    ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
    dt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[args.out_dtype]
    ob = 4 if args.out_dtype == "fp32" else 2
    at0 = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    plan0 = tw.TwPlan(ts)
    set_bytes = 2 * k * m + ob * n * m + plan0.info["wimg_bytes"]
    n_sets = max(2, int(np.ceil(2 * bench.L2_BYTES / set_bytes)) + 1)
    plans = [plan0] + [tw.TwPlan(ts) for _ in range(n_sets - 1)]
    ats = [at0] + [at0.clone() for _ in range(n_sets - 1)]
    outs = [torch.empty((n, m), dtype=dt, device="cuda") for _ in range(n_sets)]
    info = {"workload": args.workload, "out_dtype": args.out_dtype, "n_sets": n_sets,
            "algorithmic": bench.algorithmic_bytes(plan0.info, m, ob)}
    with open(os.path.join(ROOT, "gpurun_out", f"traffic_{args.workload}_{args.out_dtype}.meta.json"), "w") as f:
        json.dump(info, f)
    for i in range(args.launches):
        j = i % n_sets
        plans[j].gemm(ats[j], out=outs[j], out_dtype=dt)
    torch.cuda.synchronize()


def _num(v: str) -> float:
    return float(v.replace(",", ""))


def merge(args):
    res = {}
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    for csv_path in sorted(glob.glob(os.path.join(args.dir, "traffic_*.csv"))):
        meta_path = csv_path[:-4] + ".meta.json"
        if not os.path.exists(meta_path):
            continue
        meta = json.load(open(meta_path))
        per = {}
        with open(csv_path) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        for row in csv.DictReader(lines):
            if "tw_gemm" not in row.get("Kernel Name", "") and "tw_pair" not in row.get("Kernel Name", ""):
                continue
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(row.get("Metric Unit", "byte"), 1)
            per.setdefault(row["ID"], {})[row["Metric Name"]] = _num(row["Metric Value"]) * scale
        rd = [v["dram__bytes_read.sum"] for v in per.values() if "dram__bytes_read.sum" in v]
        wr = [v["dram__bytes_write.sum"] for v in per.values() if "dram__bytes_write.sum" in v]
        if not rd:
            continue
        key = f"{meta['workload']}:{meta['out_dtype']}"
        tot = sum(rd) / len(rd) + sum(wr) / len(wr)
        res[key] = {"bytes_per_launch": tot, "read": sum(rd) / len(rd), "write": sum(wr) / len(wr),
                    "launches": len(rd), "algorithmic": meta["algorithmic"], "ratio": tot / meta["algorithmic"],
                    "n_sets": meta["n_sets"],
                    "method": "ncu --cache-control none, single pass (no replay), rotating sets > 2x L2, "
                              "mean over the profiled launches",
                    "source": os.path.relpath(csv_path, ROOT)}
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--workload", default="C2a")
    r.add_argument("--out-dtype", default="fp16")
    r.add_argument("--launches", type=int, default=80)
    mg = sub.add_parser("merge")
    mg.add_argument("--dir", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    return run(args) if args.cmd == "run" else merge(args)


if __name__ == "__main__":
    sys.exit(main())
