"""Summarise ncu reports into profiles/ (tracked): key SOL / DRAM / tensor-pipe
metrics per kernel, plus per-launch DRAM traffic for bench.py's roofline.

    python tools/ncu_summary.py OUT.md name=gpurun_out/prof_X.ncu-rep ...
"""
import csv, io, json, os, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes (all)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (active SMs)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "warp cycles per issued inst"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, r)}
        res.append(d)
    return res


def main():
    out_md = sys.argv[1]
    lines = ["# ncu summaries (`ncu --set full --clock-control none`, one launch each, warm L2 / replayed)", ""]
    traffic = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        for d in raw(rep):
            kname = d.get("Kernel Name", ("?", ""))[0]
            lines.append(f"## {name}: `{kname[:110]}`")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for key, label in KEYS:
                if key in d:
                    v, u = d[key]
                    lines.append(f"| {label} (`{key}`) | {v} {u} |")
            lines.append("")
            if "tw_gemm" in kname and "dram__bytes_read.sum" in d:
                def to_bytes(vu):
                    v, u = vu
                    v = float(v.replace(",", ""))
                    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                traffic[name] = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    with open(tpath, "w") as f:
        json.dump(old, f, indent=1)
    print(open(out_md).read())


if __name__ == "__main__":
    main()
