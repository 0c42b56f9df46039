"""Generate golden fixtures by importing the REAL reference package.

Run here (the container that has /root/reference); the outputs are committed
under tests/golden/ so the GPU box, which has no /root/reference, can check
against them.  Nothing at test time imports the reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Fixtures:
  golden_masks.npz     mask-word KATs (pattern.py:169-189) for the lengths the
                       reference tests use (test_pattern.py:114-120) + random
  golden_patterns.npz  random_uniform_pattern(K,N,G,s,42) for every BASELINE
                       config (col_ids, mask words, pruned columns, stats)
  golden_small.npz     small end-to-end cases: bf16-rounded A/W, the
                       reference's compact() sub-matrices, gemm_tw, gemm_dense
                       (zero-fill oracle), spmm_csc / gemm_tew outputs
  golden_hashes.json   SHA-256 of full-size reference gemm_tw / gemm_tew
                       outputs at BASELINE shapes (pins the C oracle bit-exactly)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import tilewise as tw  # noqa: E402  (the reference, read-only)
from oracle.oracle import bf16_round  # noqa: E402

PATTERN_CONFIGS = {
    # name: (K, N, G, s)
    "C1": (1024, 1024, 128, 0.50),
    "C2a": (768, 3072, 128, 0.75),
    "C2b": (768, 768, 128, 0.75),
    "C4": (768, 3072, 128, 0.765),
    "C5_s0": (1024, 4096, 128, 0.0),
    "C5_s10": (1024, 4096, 128, 0.10),
    "C5_s25": (1024, 4096, 128, 0.25),
    "C5_s50": (1024, 4096, 128, 0.50),
    "C5_s75": (1024, 4096, 128, 0.75),
    "C5_s90": (1024, 4096, 128, 0.90),
    "VGG_conv1_2_s75": (576, 64, 128, 0.75),
    "VGG_conv4_2_s50": (4608, 512, 128, 0.50),
    "VGG_conv5_1_s75": (4608, 512, 128, 0.75),
    "G64_s60": (256, 256, 64, 0.60),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def flat_pattern(p):
    cols = np.concatenate([t.col_ids for t in p.tiles]).astype(np.int32) if p.tiles else np.zeros(0, np.int32)
    n_i = np.array([t.n_i for t in p.tiles], np.int32)
    words = np.stack([tw.pattern.pack_mask_words(t.row_keep) for t in p.tiles]) if p.tiles else np.zeros((0, 1), np.uint32)
    return cols, n_i, words


def gen_masks(out):
    rng = np.random.default_rng(7)
    d = {}
    for length in (1, 31, 32, 33, 96, 100, 768, 1000):
        keep = rng.random(length) > 0.5
        d[f"keep_{length}"] = keep
        d[f"words_{length}"] = tw.pattern.pack_mask_words(keep)
        d[f"idx_{length}"] = tw.pattern.mask_words_to_indices(d[f"words_{length}"], length)
    np.savez_compressed(out, **d)


def gen_patterns(out):
    d = {}
    for name, (k, n, g, s) in PATTERN_CONFIGS.items():
        p = tw.random_uniform_pattern(k, n, g, s, seed=42)
        cols, n_i, words = flat_pattern(p)
        st = tw.pattern_stats(p, m=1)
        d[f"{name}__dims"] = np.array([k, n, g], np.int64)
        d[f"{name}__s"] = np.array([s])
        d[f"{name}__cols"] = cols
        d[f"{name}__n_i"] = n_i
        d[f"{name}__words"] = words
        d[f"{name}__k_i"] = np.array([t.k_i for t in p.tiles], np.int32)
        d[f"{name}__pruned"] = np.setdiff1d(np.arange(n), p.surviving_columns).astype(np.int64)
        d[f"{name}__sparsity"] = np.array([st.sparsity])
    np.savez_compressed(out, **d)


def small_cases():
    """(name, M, K, N, G, s, seed, kind) -- kinds exercise the edge cases the
    reference tests pin (test_engine.py:111-136, test_acceptance.py:63-81)."""
    cases = []
    rng = np.random.default_rng(1001)
    for i in range(12):
        m, k, n = (int(rng.integers(48, 200)) for _ in range(3))
        g = int((32, 64, 128)[rng.integers(3)])
        s = float((0.0, 0.25, 0.5, 0.75, 0.9)[rng.integers(5)])
        cases.append((f"rand{i}", m, k, n, g, s, 2000 + i, "random"))
    cases += [
        ("dense_g8", 16, 24, 32, 8, 0.0, 27, "dense"),
        ("g64_s60", 256, 256, 256, 64, 0.6, 35, "random"),
        ("g16_s50", 64, 96, 80, 16, 0.5, 38, "random"),
        ("dead_tile", 4, 8, 8, 4, 0.0, 29, "dead_tile"),
        ("all_pruned", 4, 8, 8, 8, 0.0, 31, "all_pruned"),
        ("g256_s50", 130, 200, 600, 256, 0.5, 77, "random"),
        ("m_ragged", 77, 130, 300, 128, 0.75, 78, "random"),
        ("k_tiny", 200, 27, 64, 128, 0.5, 79, "random"),
    ]
    return cases


def make_pattern(kind, k, n, g, s, seed):
    if kind == "dense":
        return tw.dense_pattern(k, n, g)
    if kind == "dead_tile":
        dead = tw.Tile(np.arange(8, dtype=np.int32)[4:], np.zeros(8, dtype=bool))
        live = tw.Tile(np.arange(4, dtype=np.int32), np.ones(8, dtype=bool))
        return tw.TilePattern(8, 8, 4, (live, dead))
    if kind == "all_pruned":
        return tw.TilePattern(8, 8, 8, (tw.Tile(np.arange(8, dtype=np.int32), np.zeros(8, bool)),))
    return tw.random_uniform_pattern(k, n, g, s, seed=seed)


def gen_small(out):
    d = {}
    names = []
    for name, m, k, n, g, s, seed, kind in small_cases():
        rng = np.random.default_rng(seed)
        a = bf16_round(rng.standard_normal((m, k)).astype(np.float32))
        w = bf16_round(rng.standard_normal((k, n)).astype(np.float32))
        p = make_pattern(kind, k, n, g, s, seed)
        A = tw.DenseMatrix.from_array(a)
        W = tw.DenseMatrix.from_array(w)
        ts = tw.compact(W, p)
        got = tw.gemm_tw(A, ts)
        dense = tw.gemm_dense(A, tw.zero_fill(W, p))
        cols, n_i, words = flat_pattern(p)
        d[f"{name}__dims"] = np.array([m, k, n, g], np.int64)
        d[f"{name}__seed"] = np.array([seed], np.int64)     # A, W regenerate from seed
        d[f"{name}__aw_sha256"] = np.array([sha(a) + sha(w)])
        d[f"{name}__cols"] = cols
        d[f"{name}__n_i"] = n_i
        d[f"{name}__words"] = words
        d[f"{name}__subs"] = (np.concatenate([t.sub_matrix.data for t in ts.tiles])
                              if ts.tiles else np.zeros(0, np.float32))
        d[f"{name}__ct"] = got.data.reshape(n, m)          # COL_MAJOR buffer == C^T
        # the zero-fill dense oracle is bit-identical to gemm_tw (engine.py:155-156)
        d[f"{name}__dense_bitexact"] = np.array([np.array_equal(dense.data, got.data)])
        d[f"{name}__pruned"] = np.setdiff1d(np.arange(n), p.surviving_columns).astype(np.int64)
        # TEW overlay + spmm (test_engine.py:216-230 recipe) where it applies
        st = tw.pattern_stats(p, m=1).sparsity
        if kind == "random" and st > 0.05:
            delta = min(0.015, st / 2)
            _, csc = tw.tew_overlay(W, tw.magnitude_scores(W), p,
                                    tw.TewConfig(alpha=st - delta, delta=delta))
            d[f"{name}__csc_col_ptr"] = csc.col_ptr
            d[f"{name}__csc_row_idx"] = csc.row_idx
            d[f"{name}__csc_values"] = csc.values
            d[f"{name}__delta"] = np.array([delta])
            d[f"{name}__spmm_ct"] = tw.spmm_csc(A, csc).data.reshape(n, m)
            d[f"{name}__tew_ct"] = tw.gemm_tew(A, ts, csc).data.reshape(n, m)
        names.append(name)
    d["names"] = np.array(names)
    np.savez_compressed(out, **d)


def gen_hashes(out):
    """Full-size outputs at BASELINE shapes; inputs as in cli._bench_one
    (cli.py:408-412), bf16-rounded (RNE) and held as fp32."""
    res = {}
    for name, (m, k, n, g, s) in {
        "C1": (1024, 1024, 1024, 128, 0.5),
        "C2b": (4096, 768, 768, 128, 0.75),
        "C2a": (4096, 768, 3072, 128, 0.75),
    }.items():
        rng = np.random.default_rng(42)
        a = bf16_round(rng.standard_normal((m, k)).astype(np.float32))
        w = bf16_round(rng.standard_normal((k, n)).astype(np.float32))
        p = tw.random_uniform_pattern(k, n, g, s, seed=42)
        t0 = time.perf_counter()
        ct = tw.gemm_tw(tw.DenseMatrix.from_array(a), tw.compact(tw.DenseMatrix.from_array(w), p))
        dt = time.perf_counter() - t0
        res[name] = {"dims": [m, k, n, g, s], "gemm_tw_sha256": sha(ct.data),
                     "ref_seconds_1worker": dt}
        print(name, res[name], flush=True)
    # TEW C4: 76.5% TW + 1.5% EW overlay, magnitude scores
    m, k, n, g, s = 4096, 768, 3072, 128, 0.765
    rng = np.random.default_rng(42)
    a = bf16_round(rng.standard_normal((m, k)).astype(np.float32))
    w = bf16_round(rng.standard_normal((k, n)).astype(np.float32))
    p = tw.random_uniform_pattern(k, n, g, s, seed=42)
    W = tw.DenseMatrix.from_array(w)
    sp = tw.pattern_stats(p, m=1).sparsity
    _, csc = tw.tew_overlay(W, tw.magnitude_scores(W), p, tw.TewConfig(alpha=sp - 0.015, delta=0.015))
    ts = tw.compact(W, p)
    ct = tw.gemm_tew(tw.DenseMatrix.from_array(a), ts, csc)
    h = hashlib.sha256()
    for arr in (csc.col_ptr, csc.row_idx, csc.values):
        h.update(np.ascontiguousarray(arr).tobytes())
    res["C4"] = {"dims": [m, k, n, g, s], "delta": 0.015, "nnz": int(csc.nnz),
                 "csc_sha256": h.hexdigest(), "gemm_tew_sha256": sha(ct.data)}
    print("C4", res["C4"], flush=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    gen_masks(os.path.join(HERE, "golden_masks.npz"))
    gen_patterns(os.path.join(HERE, "golden_patterns.npz"))
    gen_small(os.path.join(HERE, "golden_small.npz"))
    gen_hashes(os.path.join(HERE, "golden_hashes.json"))
    print("done")
