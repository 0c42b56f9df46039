"""PCIe copy shapes of the e2e path: 1-D pinned D2H vs the 2-D (strided) D2H of
token chunks that _gemm_tw_pipelined issues, and the e2e call itself by chunk."""
import os, statistics, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2008_13006_b200 import _lib

def timed(fn, reps=7):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3

n, m = 3072, 4096
dev = torch.empty((n, m), dtype=torch.float32, device="cuda")
host = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
s = torch.cuda.current_stream().cuda_stream
print("1-D D2H 50 MB: %.3f ms" % timed(lambda: host.copy_(dev, non_blocking=True)))
for ch in (512, 1024, 2048, 4096):
    def f():
        for c0 in range(0, m, ch):
            _lib.call("tw_copy_2d", host.data_ptr() + c0 * 4, m * 4, dev.data_ptr() + c0 * 4, m * 4, ch * 4, n, 1, s)
    print("2-D D2H in %d-token chunks: %.3f ms" % (ch, timed(f)))
