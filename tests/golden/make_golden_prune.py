"""prune_stage fixtures written by the REAL reference (pruning.py:262-335,
the step before the TW path).  Run here, where
/root/reference exists; the small npz is committed and read back by
tests/test_prune.py (no reference at test time).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_prune.py
"""
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402

import tilewise as ref  # noqa: E402  (the reference, read-only)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_prune.npz")
rng = np.random.default_rng(11)
cases = []
# (K, N, G, s_t, scores kind, staged): magnitude and heterogeneous scores,
# a G=64 case with a remainder tile, a two-stage run (prev), and ties
for i, (k, n, g, s_t, kind, staged) in enumerate([
        (64, 200, 32, 0.5, "mag", False), (96, 150, 64, 0.6, "het", False),
        (128, 384, 128, 0.75, "mag", True), (40, 70, 16, 0.3, "ties", False),
        (160, 320, 64, 0.9, "het", True), (8, 9, 4, 0.5, "ties", True)]):
    w = rng.standard_normal((k, n)).astype(np.float32)
    if kind == "het":  # gamma row/column scales: units differ systematically
        w *= rng.gamma(2.0, 1.0, (k, 1)).astype(np.float32) * rng.gamma(2.0, 1.0, (1, n)).astype(np.float32)
    wd = ref.DenseMatrix.from_array(w)
    if kind == "ties":  # quantised magnitudes: many equal unit scores
        sm = ref.ScoreMap(np.round(np.abs(w.astype(np.float64)) * 2) / 2)
    else:
        sm = ref.magnitude_scores(wd)
    prev = ref.prune_stage(wd, sm, s_t * 0.6, g) if staged else None
    p = ref.prune_stage(wd, sm, s_t, g, prev=prev)
    # scores are rebuilt from w (float32) and the kind: |w| in float64, or
    # round(2|w|)/2 for "ties" (keeps the fixture small)
    rec = {"k": k, "n": n, "g": g, "s_t": s_t, "w": w, "ties": int(kind == "ties"), "staged": int(staged)}
    for tag, pat in (("prev", prev), ("out", p)):
        if pat is None:
            continue
        rec[f"{tag}_cols"] = np.concatenate([t.col_ids for t in pat.tiles]).astype(np.int32) if pat.tiles else np.zeros(0, np.int32)
        rec[f"{tag}_off"] = np.cumsum([0] + [t.col_ids.size for t in pat.tiles]).astype(np.int64)
        rec[f"{tag}_keep"] = (np.stack([t.row_keep for t in pat.tiles]) if pat.tiles else np.zeros((0, k), bool))
    rec["prev_s_t"] = s_t * 0.6
    cases.append(rec)
flat = {}
for i, c in enumerate(cases):
    for key, v in c.items():
        flat[f"c{i}_{key}"] = np.asarray(v)
flat["n_cases"] = np.asarray(len(cases))
np.savez_compressed(OUT, **flat)
print("wrote", OUT, len(cases), "cases")
