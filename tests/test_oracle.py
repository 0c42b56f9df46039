"""Pin the CPU oracle (oracle/) against the golden fixtures generated from the
real reference (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import oracle as orc
from tests import golden_io as gio


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


@pytest.mark.parametrize("length", [1, 31, 32, 33, 96, 100, 768, 1000])
def test_mask_words_match_reference(length):
    d = gio.load("golden_masks.npz")
    keep = d[f"keep_{length}"]
    words = orc.pack_mask_words(keep)
    assert words.dtype == np.uint32
    assert np.array_equal(words, d[f"words_{length}"])
    assert np.array_equal(orc.unpack_mask_words(words, length), keep)
    assert np.array_equal(orc.mask_words_to_indices(words, length), d[f"idx_{length}"])


def test_pattern_generator_matches_reference():
    d = gio.load("golden_patterns.npz")
    names = sorted({k.split("__")[0] for k in d})
    assert len(names) >= 10
    for name in names:
        k, n, g = (int(x) for x in d[f"{name}__dims"])
        s = float(d[f"{name}__s"][0])
        p = orc.random_uniform_pattern(k, n, g, s, 42)
        cols = np.concatenate([c for c, _ in p[3]]) if p[3] else np.zeros(0, np.int32)
        assert np.array_equal(cols, d[f"{name}__cols"]), name
        assert np.array_equal(np.array([c.size for c, _ in p[3]]), d[f"{name}__n_i"]), name
        words = np.stack([orc.pack_mask_words(kp) for _, kp in p[3]])
        assert np.array_equal(words, d[f"{name}__words"]), name
        assert np.array_equal(orc.pruned_columns(p), d[f"{name}__pruned"]), name
        _, _, sp = orc.pattern_flops(p, 1)
        assert sp == float(d[f"{name}__sparsity"][0]), name


@pytest.mark.parametrize("name", gio.small_names())
def test_oracle_small_cases_bitexact(name):
    c = gio.small_case(name)
    assert sha(c["a"]) + sha(c["w"]) == c["aw_sha256"], "input regeneration drifted"
    tiles = orc.compact(c["w"], c["pattern"])
    subs = np.concatenate([np.ravel(t.sub, order="F") for t in tiles]) if tiles else np.zeros(0, np.float32)
    assert np.array_equal(subs, c["subs"])
    assert np.array_equal(orc.pruned_columns(c["pattern"]), c["pruned"])
    packed = orc.PackedTiles(tiles, c["k"], c["n"])
    at = np.ascontiguousarray(c["a"].T)
    ct = orc.gemm_tw_ct(at, packed, threads=1)
    assert np.array_equal(ct, c["ct"])
    ct4 = orc.gemm_tw_ct(at, packed, threads=4)
    assert np.array_equal(ct4, c["ct"])
    dense = orc.gemm_dense_ct(at, orc.zero_fill(c["w"], c["pattern"]))
    assert np.array_equal(dense, c["ct"]) == c["dense_bitexact"]
    if "csc" in c:
        cp, ri, va = c["csc"]
        mine = orc.tew_overlay_magnitude(c["w"], c["pattern"], c["delta"])
        assert all(np.array_equal(x, y) for x, y in zip(mine, c["csc"]))
        assert np.array_equal(orc.spmm_csc_ct(at, cp, ri, va), c["spmm_ct"])
        assert np.array_equal(orc.gemm_tew_ct(at, packed, cp, ri, va), c["tew_ct"])


def test_naive_python_loop_agrees_with_c_oracle():
    c = gio.small_case("g16_s50")
    tiles = orc.compact(c["w"], c["pattern"])
    at = np.ascontiguousarray(c["a"].T)
    assert np.array_equal(orc.naive_gemm_tw_ct(at, tiles, c["n"]), c["ct"])


@pytest.mark.parametrize("name", ["C1", "C2b", "C2a"])
def test_oracle_full_size_hash_matches_reference(name):
    h = gio.load("golden_hashes.json")[name]
    m, k, n, g, s = h["dims"]
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
    packed = orc.PackedTiles(orc.compact(w, p), k, n)
    ct = orc.gemm_tw_ct(np.ascontiguousarray(a.T), packed, threads=orc.max_threads())
    assert sha(ct) == h["gemm_tw_sha256"]


SHAPE_CASES = ["C5_s0", "C5_s75", "C5_s90", "VGG_conv1_1_s50", "VGG_conv1_2_s75", "VGG_conv4_2_s50", "NMT_lstm_s75"]


@pytest.mark.parametrize("name", SHAPE_CASES)
def test_oracle_baseline_shapes_hash_matches_reference(name):
    """C5 BERT-large, VGG-16 im2col and the NMT LSTM gate shape (reduced M):
    the C oracle reproduces the reference's gemm_tw bit for bit
    (tests/golden/make_golden_shapes.py), and the oracle pattern generator
    reproduces the reference's tile structure."""
    h = gio.load("golden_hashes_shapes.json")[name]
    m, k, n, g, s = h["dims"]
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
    tiles = p[3]
    assert len(tiles) == h["tiles"]
    assert [len(c) for c, _ in tiles] == h["n_i"]
    assert sorted({int(keep.sum()) for _, keep in tiles}) == h["k_i"]
    assert len(orc.pruned_columns(p)) == h["pruned_columns"]
    packed = orc.PackedTiles(orc.compact(w, p), k, n)
    ct = orc.gemm_tw_ct(np.ascontiguousarray(a.T), packed, threads=orc.max_threads())
    assert sha(ct) == h["gemm_tw_sha256"]


def test_oracle_tew_full_size_hash_matches_reference():
    h = gio.load("golden_hashes.json")["C4"]
    m, k, n, g, s = h["dims"]
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)
    sp = orc.pattern_flops(p, 1)[2]
    assert abs(sp - s) < 0.01
    cp, ri, va = orc.tew_overlay_magnitude(w, p, h["delta"])
    assert int(cp[-1]) == h["nnz"]
    hh = hashlib.sha256()
    for arr in (cp, ri, va):
        hh.update(np.ascontiguousarray(arr).tobytes())
    assert hh.hexdigest() == h["csc_sha256"]
    packed = orc.PackedTiles(orc.compact(w, p), k, n)
    ct = orc.gemm_tew_ct(np.ascontiguousarray(a.T), packed, cp, ri, va, threads=orc.max_threads())
    assert sha(ct) == h["gemm_tew_sha256"]


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(3).standard_normal(100000).astype(np.float32) * 100
    x[:4] = [0.0, -0.0, 1e-40, -3.3895314e38]
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(orc.bf16_round(x), want)
