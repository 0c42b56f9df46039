"""Where the e2e gemm_tw call's time goes beyond the PCIe floor (C2a, host fp32 in/out):
the whole call, the host time until the call has enqueued everything, and a
transfer-only pipeline (the same H2D / 2-D D2H chunks without prep/GEMM)."""
import os, statistics, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2008_13006_b200 as tw
from paper_2008_13006_b200 import _lib, engine
from oracle import oracle as orc

m, k, n, g, s, _ = bench.WORKLOADS["C2a"]
a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
a_pin = torch.empty(m * k, dtype=torch.float32, pin_memory=True)
a_pin.copy_(torch.from_numpy(a.reshape(-1)))
a_host = tw.DenseMatrix(m, k, tw.Layout.ROW_MAJOR, a_pin.numpy())
c_pin = torch.empty(m * n, dtype=torch.float32, pin_memory=True).numpy()

def med(fn, reps=30):
    for _ in range(5): fn()
    ts_ = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts_.append(time.perf_counter() - t0)
    return statistics.median(ts_) * 1e3

for ch in (1024, 2048, 4096):
    engine._PIPE_CHUNK = ch
    t_call = med(lambda: tw.gemm_tw(a_host, ts, out=c_pin, precision="bf16"))
    print(f"chunk {ch}: e2e call {t_call:.3f} ms")
engine._PIPE_CHUNK = 1024
# host-side cost: profile one call
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable()
for _ in range(20): tw.gemm_tw(a_host, ts, out=c_pin, precision="bf16")
pr.disable()
st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats("tottime").print_stats(12); print(st.getvalue()[:3000])
# transfer-only pipeline
a_dev = torch.empty((m, k), dtype=torch.float32, device="cuda")
ct = torch.empty((n, m), dtype=torch.float32, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
a_t = torch.from_numpy(a_pin.numpy()).view(m, k)
def xfer(ch=1024):
    cur = torch.cuda.current_stream()
    for c0 in range(0, m, ch):
        with torch.cuda.stream(s_in):
            a_dev[c0:c0 + ch].copy_(a_t[c0:c0 + ch], non_blocking=True)
        cur.wait_stream(s_in)
        s_out.wait_stream(cur)
        _lib.call("tw_copy_2d", c_pin.ctypes.data + c0 * 4, m * 4, ct.data_ptr() + c0 * 4, m * 4, ch * 4, n, 1, s_out.cuda_stream)
    s_out.synchronize()
print("transfer-only pipeline (1024-token chunks): %.3f ms" % med(xfer))
