"""Top stalled SASS instructions of an ncu report: python tools/sass_hot.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
iall, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
print("total samples", sum(int(r[iall] or 0) for r in data))
for r in sorted(data, key=lambda r: -int(r[iall] or 0))[:n]:
    st = sorted([(float(r[i] or 0), h[i][6:]) for i in stall], reverse=True)[:2]
    print(f"{r[ia][-5:]} {r[iall]:>5} {r[iex]:>8}  {r[isrc][:58]:58s} {[(k, int(v)) for v, k in st if v > 0]}")
