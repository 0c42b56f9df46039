"""Binary format fixtures written by the REAL reference (TWPT / TWCS / TWMX,
pattern.py:373-420, matrix.py:207-283).  Run here, where
/root/reference exists; the small files under tests/golden/fmt/ are
committed and read back by tests/test_formats.py (no reference at test time).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_formats.py
"""
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402

import tilewise as ref  # noqa: E402  (the reference, read-only)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fmt")
os.makedirs(OUT, exist_ok=True)
rng = np.random.default_rng(7)
# patterns: BERT-base attention-out (C2b) and a G=64 case with a remainder tile
ref.write_pattern(ref.random_uniform_pattern(768, 768, 128, 0.75, seed=42), os.path.join(OUT, "c2b.twpt"))
ref.write_pattern(ref.random_uniform_pattern(96, 150, 64, 0.6, seed=3), os.path.join(OUT, "g64.twpt"))
# dense weights (row- and col-major) matching the G=64 pattern
w = rng.standard_normal((96, 150)).astype(np.float32)
ref.write_matrix(ref.DenseMatrix.from_array(w), os.path.join(OUT, "w_g64.twmx"))
ref.write_matrix(ref.DenseMatrix.from_array(w, ref.Layout.COL_MAJOR), os.path.join(OUT, "w_g64_col.twmx"))
# TEW overlay for the same weights/pattern
p = ref.random_uniform_pattern(96, 150, 64, 0.6, seed=3)
wd = ref.DenseMatrix.from_array(w)
sp = ref.pattern_stats(p, m=1).sparsity
_, ew = ref.tew_overlay(wd, ref.magnitude_scores(wd), p, ref.TewConfig(alpha=sp - 0.02, delta=0.02))
ref.write_csc(ew, os.path.join(OUT, "ew_g64.twcs"))
for f in sorted(os.listdir(OUT)):
    print(f, os.path.getsize(os.path.join(OUT, f)))
# a 2-layer TWML checkpoint + its pattern_<i>.twpt files (the `verify` CLI input)
rng2 = np.random.default_rng(9)
model = ref.MlpModel([rng2.standard_normal((64, 96)) * 0.2, rng2.standard_normal((96, 10)) * 0.2],
                     [rng2.standard_normal(96) * 0.1, rng2.standard_normal(10) * 0.1])
ref.save_model(model, os.path.join(OUT, "mlp.twml"))
ref.write_pattern(ref.random_uniform_pattern(64, 96, 32, 0.5, seed=1), os.path.join(OUT, "pattern_0.twpt"))
ref.write_pattern(ref.random_uniform_pattern(96, 10, 8, 0.5, seed=2), os.path.join(OUT, "pattern_1.twpt"))
print("mlp.twml", os.path.getsize(os.path.join(OUT, "mlp.twml")))
