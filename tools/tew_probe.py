"""Time the pieces of gemm_tew at C4 (TEW on BERT-base FC1): SpMM alone,
TW accumulate alone, TW overwrite, and the composite."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench, paper_2008_13006_b200 as tw
from oracle import oracle as orc
from tools.sweep import timed

m, k, n = 4096, 768, 3072
rng = np.random.default_rng(42)
w = orc.bf16_round(rng.standard_normal((k, n)).astype(np.float32))
p = orc.random_uniform_pattern(k, n, 128, 0.765, 42)
ts = tw.compact(tw.DenseMatrix.from_array(w), bench.to_pattern(tw, p))
plan = tw.TwPlan(ts)
cp, ri, va = orc.tew_overlay_magnitude(w, p, 0.015)
csc = tw.DeviceCsc(tw.CscMatrix(k, n, cp, ri, va))
at = torch.randn((k, m), device="cuda").to(torch.bfloat16)
out = torch.empty((n, m), device="cuda")
out16 = torch.empty((n, m), device="cuda", dtype=torch.float16)
for name, fn in [("spmm overwrite", lambda i: tw.spmm_csc_device(at, csc, out=out)),
                 ("spmm accumulate", lambda i: tw.spmm_csc_device(at, csc, out=out, accumulate=True)),
                 ("tw overwrite", lambda i: plan.gemm(at, out=out)),
                 ("tw accumulate", lambda i: plan.gemm(at, out=out, accumulate=True)),
                 ("gemm_tew (TW + SpMM)", lambda i: plan.gemm_tew(at, csc, out=out, merged=False)),
                 ("gemm_tew (merged plan)", lambda i: plan.gemm_tew(at, csc, out=out)),
                 ("gemm_tew merged fp16", lambda i: plan.gemm_tew(at, csc, out=out16, out_dtype=torch.float16))]:
    print(f"{name:24s} {timed(fn, 20):8.1f} us", flush=True)
print("nnz", csc.nnz)
