"""Loaders for the committed golden fixtures (tests/golden/, generated from the
real reference by tests/golden/make_golden.py)."""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_cache: dict = {}


def load(name: str):
    if name not in _cache:
        path = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            with open(path) as f:
                _cache[name] = json.load(f)
        else:
            _cache[name] = dict(np.load(path, allow_pickle=False))
    return _cache[name]


def pattern_from(d: dict, prefix: str, k: int, n: int, g: int):
    """Rebuild the oracle's tuple pattern (k, n, g, [(cols, keep)]) from a
    flattened fixture."""
    from oracle.oracle import unpack_mask_words

    cols = d[f"{prefix}__cols"]
    n_i = d[f"{prefix}__n_i"]
    words = d[f"{prefix}__words"]
    tiles = []
    off = 0
    for t in range(n_i.size):
        c = cols[off: off + n_i[t]].astype(np.int32)
        off += int(n_i[t])
        tiles.append((c, unpack_mask_words(words[t], k)))
    return (k, n, g, tiles)


def small_names():
    return [str(x) for x in load("golden_small.npz")["names"]]


def small_case(name: str):
    """-> dict(m,k,n,g, a, w, pattern, ct, pruned, subs, [csc..])"""
    d = load("golden_small.npz")
    m, k, n, g = (int(x) for x in d[f"{name}__dims"])
    seed = int(d[f"{name}__seed"][0])
    from oracle.oracle import bf16_round

    rng = np.random.default_rng(seed)
    a = bf16_round(rng.standard_normal((m, k)).astype(np.float32))
    w = bf16_round(rng.standard_normal((k, n)).astype(np.float32))
    out = dict(m=m, k=k, n=n, g=g, a=a, w=w,
               pattern=pattern_from(d, name, k, n, g),
               ct=d[f"{name}__ct"], pruned=d[f"{name}__pruned"], subs=d[f"{name}__subs"],
               aw_sha256=str(d[f"{name}__aw_sha256"][0]),
               dense_bitexact=bool(d[f"{name}__dense_bitexact"][0]))
    if f"{name}__csc_col_ptr" in d:
        out.update(csc=(d[f"{name}__csc_col_ptr"], d[f"{name}__csc_row_idx"], d[f"{name}__csc_values"]),
                   delta=float(d[f"{name}__delta"][0]),
                   spmm_ct=d[f"{name}__spmm_ct"], tew_ct=d[f"{name}__tew_ct"])
    return out
