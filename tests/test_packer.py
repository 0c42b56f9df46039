"""Host-side packer (north_star item 1) -- CPU only.  Bit-exact against the
golden fixtures from the reference and against the oracle's restatement:
mask words, kept-K index lists, compacted sub-matrices, pruned-column lists,
and the packed plan image the sm_100a kernel consumes."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2008_13006_b200 as tw
from paper_2008_13006_b200 import _lib
from oracle import oracle as orc
from tests import golden_io as gio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tw_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tw_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert L.tw_version() >= 100


def to_tw_pattern(p):
    k, n, g, tiles = p
    return tw.TilePattern(k, n, g, tuple(tw.Tile(c, keep) for c, keep in tiles))


@pytest.mark.parametrize("length", [1, 31, 32, 33, 96, 100, 768, 1000])
def test_mask_words_bitexact(length):
    d = gio.load("golden_masks.npz")
    keep = d[f"keep_{length}"]
    words = tw.pack_mask_words(keep)
    assert words.dtype == np.uint32 and np.array_equal(words, d[f"words_{length}"])
    assert np.array_equal(tw.unpack_mask_words(words, length), keep)
    assert np.array_equal(tw.mask_words_to_indices(words, length), d[f"idx_{length}"])


def test_unpack_too_short_raises_dimension_error():
    with pytest.raises(tw.DimensionError):
        tw.unpack_mask_words(np.zeros(1, np.uint32), 33)


def test_random_uniform_pattern_matches_reference():
    d = gio.load("golden_patterns.npz")
    for name in sorted({k.split("__")[0] for k in d}):
        k, n, g = (int(x) for x in d[f"{name}__dims"])
        p = tw.random_uniform_pattern(k, n, g, float(d[f"{name}__s"][0]), 42)
        assert np.array_equal(p.surviving_columns, d[f"{name}__cols"]), name
        assert [t.k_i for t in p.tiles] == list(d[f"{name}__k_i"]), name
        assert np.array_equal(tw.pruned_columns(p), d[f"{name}__pruned"]), name
        assert tw.pattern_stats(p, 1).sparsity == float(d[f"{name}__sparsity"][0])


@pytest.mark.parametrize("name", gio.small_names())
def test_compact_bitexact_vs_reference(name):
    c = gio.small_case(name)
    p = to_tw_pattern(c["pattern"])
    for layout in (tw.Layout.ROW_MAJOR, tw.Layout.COL_MAJOR):
        w = tw.DenseMatrix.from_array(c["w"], layout)
        ts = tw.compact(w, p)
        subs = np.concatenate([t.sub_matrix.data for t in ts.tiles]) if ts.tiles else np.zeros(0, np.float32)
        assert np.array_equal(subs, c["subs"])
        for t, ref in zip(ts.tiles, p.tiles):
            assert t.sub_matrix.layout == tw.Layout.COL_MAJOR
            assert np.array_equal(t.row_mask_words, orc.pack_mask_words(ref.row_keep))
        assert np.array_equal(ts.expand().array(), tw.zero_fill(w, p).array())
    assert np.array_equal(tw.pruned_columns(p), c["pruned"])


def decode_wimg(img: np.ndarray, wrows: int, nkb: int, n_i: int, k_i: int, dtype=np.uint16):
    """Undo the SW128 swizzle of one tile's weight image -> (k_pad x wrows)."""
    blk = img.view(np.uint16).reshape(nkb, wrows, 8, 8)  # kb, row j, phys chunk, elem
    out = np.zeros((nkb * 64, wrows), np.uint16)
    for j in range(wrows):
        for c in range(8):
            out[np.arange(nkb)[:, None] * 64 + c * 8 + np.arange(8)[None, :], j] = blk[:, j, c ^ (j & 7), :]
    return out


def bf16_bits(x: np.ndarray) -> np.ndarray:
    return (orc.bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("name", ["g64_s60", "m_ragged", "g256_s50", "dead_tile", "all_pruned", "k_tiny", "rand3"])
def test_packed_plan_image_bitexact(name):
    c = gio.small_case(name)
    p = to_tw_pattern(c["pattern"])
    ts = tw.compact(tw.DenseMatrix.from_array(c["w"]), p)
    pl = tw.PackedPlan(ts, "bf16")
    k = c["k"]
    table = pl.export("tiles")
    kidx, colids, zero, wimg = pl.export("kidx"), pl.export("colids"), pl.export("zero_rows"), pl.export("wimg")
    bn = pl.info["block_n"]
    live = [i for i, t in enumerate(p.tiles) if t.k_i > 0]
    assert sorted(table[:, 0].tolist()) == live
    # LPT order: non-increasing k_i * n_i
    work = table[:, 4] * table[:, 3]
    assert all(work[i] >= work[i + 1] for i in range(len(work) - 1))
    wrows = (wimg.size // max(int(table[:, 6].sum()), 1)) // 128 if len(table) else 0
    for src, koff, coff, n_i, k_i, k16, nkb, woff in table:
        t = p.tiles[src]
        rows = np.flatnonzero(t.row_keep)
        assert k_i == rows.size and n_i == t.n_i
        assert k16 == (k_i + 15) // 16 and nkb == (k_i + 63) // 64
        lst = kidx[koff: koff + nkb * 64]
        assert np.array_equal(lst[:k_i], rows) and np.all(lst[k_i:] == k)  # pad = K -> TMA OOB zero fill
        assert np.array_equal(colids[coff: coff + n_i], t.col_ids)
        assert np.all(colids[coff + n_i: coff + bn] == -1)
        dec = decode_wimg(wimg[woff: woff + nkb * wrows * 128], wrows, nkb, n_i, k_i)
        want = np.zeros_like(dec)
        want[:k_i, :n_i] = bf16_bits(ts.tiles[src].sub_matrix.array())
        assert np.array_equal(dec, want)
    dead_cols = np.concatenate([t.col_ids for t in p.tiles if t.k_i == 0] + [np.zeros(0, np.int32)])
    assert np.array_equal(np.sort(zero), np.union1d(c["pruned"], dead_cols))
    assert pl.info["kept_elems"] == sum(t.k_i * t.n_i for t in p.tiles)


def test_packed_plan_shards_partition_the_columns():
    a, w, p = orc.bench_inputs(64, 256, 1000, 128, 0.5, seed=5)
    pt = to_tw_pattern(p)
    ts = tw.compact(tw.DenseMatrix.from_array(w), pt)
    full = tw.PackedPlan(ts)
    bounds = [0, 250, 500, 750, 1000]
    kept = 0
    seen = []
    for c0, c1 in zip(bounds, bounds[1:]):
        sh = tw.PackedPlan(ts, col_range=(c0, c1))
        kept += sh.info["kept_elems"]
        table, colids = sh.export("tiles"), sh.export("colids")
        for row in table:
            ids = colids[row[2]: row[2] + row[3]] + c0
            assert np.all((ids >= c0) & (ids < c1))
            seen.append(ids)
        z = sh.export("zero_rows") + c0
        assert np.all((z >= c0) & (z < c1))
        seen.append(z)
    allc = np.sort(np.concatenate(seen))
    assert np.array_equal(allc, np.arange(1000))
    assert kept == full.info["kept_elems"]


def test_fp16_plan_image():
    c = gio.small_case("g16_s50")
    ts = tw.compact(tw.DenseMatrix.from_array(c["w"]), to_tw_pattern(c["pattern"]))
    pl = tw.PackedPlan(ts, "fp16")
    table, wimg = pl.export("tiles"), pl.export("wimg")
    wrows = wimg.size // int(table[:, 6].sum()) // 128
    src, _, _, n_i, k_i, _, nkb, woff = table[0]
    dec = decode_wimg(wimg[woff: woff + nkb * wrows * 128], wrows, nkb, n_i, k_i)
    want = ts.tiles[src].sub_matrix.array().astype(np.float16).view(np.uint16)
    assert np.array_equal(dec[:k_i, :n_i], want)


def test_compact_shape_mismatch_raises():
    p = tw.dense_pattern(8, 8, 8)
    with pytest.raises(tw.DimensionError):
        tw.compact(tw.DenseMatrix.from_array(np.zeros((8, 7), np.float32)), p)


def test_pattern_invariants_match_reference_errors():
    with pytest.raises(tw.DimensionError):
        tw.TilePattern(8, 8, 4, (tw.Tile(np.array([0, 1], np.int32), np.ones(8, bool)),
                                 tw.Tile(np.array([2, 3, 4, 5], np.int32), np.ones(8, bool))))
    with pytest.raises(tw.DimensionError):
        tw.TilePattern(8, 8, 4, (tw.Tile(np.array([1, 0], np.int32), np.ones(8, bool)),))
    with pytest.raises(tw.DimensionError):
        tw.TilePattern(8, 8, 4, (tw.Tile(np.array([0], np.int32), np.ones(8, bool)),
                                 tw.Tile(np.array([0], np.int32), np.ones(8, bool))))


def test_g_over_256_is_rejected():
    p = tw.dense_pattern(8, 512, 512)
    ts = tw.compact(tw.DenseMatrix.from_array(np.ones((8, 512), np.float32)), p)
    with pytest.raises(RuntimeError):
        tw.PackedPlan(ts)


def test_reference_objects_are_accepted_duck_typed():
    """A reference-side DenseMatrix-like object goes through as_dense."""
    class RefDense:  # stands in for tilewise.DenseMatrix
        def __init__(self, arr):
            self.rows, self.cols = arr.shape
            self.layout = 0
            self.data = arr.reshape(-1)
    arr = np.arange(12, dtype=np.float32).reshape(3, 4)
    from paper_2008_13006_b200.matrix import as_dense
    d = as_dense(RefDense(arr))
    assert np.array_equal(d.array(), arr)


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = gio.small_case("g16_s50")
    ts = tw.compact(tw.DenseMatrix.from_array(c["w"]), to_tw_pattern(c["pattern"]))
    with pytest.raises(Exception):
        tw.gemm_tw(tw.DenseMatrix.from_array(c["a"]), ts)


@pytest.mark.parametrize("seed,s,delta", [(1, 0.765, 0.015), (2, 0.5, 0.05), (3, 0.9, 0.002)])
def test_tew_merged_tileset_is_tw_plus_overlay(seed, s, delta):
    """gemm_tew's merged plan: expand(merged) == expand(tiles) + S exactly,
    tiles stay disjoint and <= G wide, and it packs."""
    from paper_2008_13006_b200.engine import tew_merged_tileset
    k, n, g = 200, 700, 128
    _, w, p = orc.bench_inputs(8, k, n, g, s, seed=seed)
    cp, ri, va = orc.tew_overlay_magnitude(w, p, delta)
    ts = tw.compact(tw.DenseMatrix.from_array(w), to_tw_pattern(p))
    merged = tew_merged_tileset(ts, tw.CscMatrix(k, n, cp, ri, va))
    dense_s = np.zeros((k, n), np.float32)
    dense_s[ri, np.repeat(np.arange(n), np.diff(cp))] = va
    assert np.array_equal(merged.expand().array(), ts.expand().array() + dense_s)
    cols = np.concatenate([t.col_ids for t in merged.tiles])
    assert np.unique(cols).size == cols.size and max(t.col_ids.size for t in merged.tiles) <= g
    plan = tw.PackedPlan(merged)
    assert plan.info["kept_elems"] >= ts_kept(ts)


def ts_kept(ts):
    return sum(t.sub_matrix.rows * t.sub_matrix.cols for t in ts.tiles)


def test_tew_overlay_in_product_matches_reference_hash():
    """tew_overlay / TewConfig / magnitude_scores in the product (pruning.py:
    132-159, :527-561 of the reference): the C4 overlay is bit-identical to
    the one the reference wrote (csc_sha256 from tests/golden/make_golden.py),
    and the small golden cases' overlays match the reference's arrays."""
    import hashlib

    from tests import golden_io as gio

    h = gio.load("golden_hashes.json")["C4"]
    m, k, n, g, s = h["dims"]
    _, w, p = orc.bench_inputs(m, k, n, g, s, seed=42)  # A is drawn first: same M
    pat = tw.TilePattern(k, n, g, tuple(tw.Tile(c, keep) for c, keep in p[3]))
    sp = tw.pattern_stats(pat, m=1).sparsity
    W = tw.DenseMatrix.from_array(w)
    out_p, csc = tw.tew_overlay(W, tw.magnitude_scores(W), pat, tw.TewConfig(alpha=sp - h["delta"], delta=h["delta"]))
    assert out_p is pat and csc.nnz == h["nnz"]
    hh = hashlib.sha256()
    for arr in (csc.col_ptr, csc.row_idx, csc.values):
        hh.update(np.ascontiguousarray(arr).tobytes())
    assert hh.hexdigest() == h["csc_sha256"]
    for name in gio.small_names():
        c = gio.small_case(name)
        if "csc" not in c:
            continue
        pat = tw.TilePattern(c["k"], c["n"], c["g"], tuple(tw.Tile(cc, keep) for cc, keep in c["pattern"][3]))
        sp = tw.pattern_stats(pat, m=1).sparsity
        W = tw.DenseMatrix.from_array(c["w"])
        delta = float(c["delta"])
        _, got = tw.tew_overlay(W, tw.magnitude_scores(W), pat, tw.TewConfig(alpha=sp - delta, delta=delta))
        cp, ri, va = c["csc"]
        assert np.array_equal(got.col_ptr, cp) and np.array_equal(got.row_idx, ri) and np.array_equal(got.values, va)
    with pytest.raises(tw.ConfigError):
        tw.TewConfig(alpha=0.5, delta=0.6)
    with pytest.raises(tw.ConfigError):  # sparsity far from alpha + delta
        tw.tew_overlay(W, tw.magnitude_scores(W), pat, tw.TewConfig(alpha=0.01, delta=0.01))


def test_reference_engine_task_api_names():
    """engine.py:24-81 names the drop-in exports: TileTask / BatchGroup /
    gather_rows / group_by_shape (host semantics; execute_batched runs on
    the GPU, tests/test_gpu_parity.py)."""
    rng = np.random.default_rng(4)
    at = rng.standard_normal((40, 7)).astype(np.float32)
    keep = rng.random(40) > 0.5
    words = tw.pack_mask_words(keep)
    assert np.array_equal(tw.gather_rows(at, words), at[keep])
    full = tw.pack_mask_words(np.ones(40, bool))
    assert tw.gather_rows(at, full) is at and tw.gather_rows(at, full, force_copy=True) is not at
    mk = lambda i, kk, nn: tw.TileTask(i, np.zeros((kk, 7), np.float32), np.zeros((kk, nn), np.float32, order="F"),  # noqa: E731
                                       np.arange(nn, dtype=np.int64))
    groups = tw.group_by_shape([mk(0, 4, 8), mk(1, 9, 16), mk(2, 4, 16), mk(3, 30, 8)])
    assert [g.n_i for g in groups] == [8, 16] and [t.index for t in groups[0].tasks] == [0, 3]
    assert groups[0].flops == 2 * 7 * (4 * 8 + 30 * 8)


@pytest.mark.parametrize("m,dt", [(4096, "fp16"), (140_000, "fp32"), (3_211_264, "fp16"), (802_816, "fp32")])
def test_zero_rows_scheduled_in_balanced_pieces(m, dt):
    """Zero rows (pruned output columns) are scheduled as pieces of <= 256 KB
    of one C^T row (64-token multiples, tw_schedule.cpp zero_pieces), so a
    long layer's pruned columns spread over the CTAs: the piece count is
    rows x pieces-per-row, and no CTA gets more than a couple of pieces above
    the lightest one (whole 6.4 MB rows landed on 32 of 148 CTAs before)."""
    from paper_2008_13006_b200.engine import PackedPlan

    k, n = 64, 256
    _, w, p = orc.bench_inputs(8, k, n, 128, 0.75, seed=3)
    pp = PackedPlan(tw.compact(tw.DenseMatrix.from_array(w), tw.TilePattern(k, n, 128, tuple(
        tw.Tile(c, keep) for c, keep in p[3]))))
    rows = len(orc.pruned_columns(p))
    ob = 4 if dt == "fp32" else 2
    cpr = max(1, -(-m * ob // (256 << 10)))
    chunk = -(-(-(-m // cpr)) // 64) * 64
    cpr = max(1, -(-m // chunk))
    units, uoff, zoff = pp.schedule(m, dt)
    assert zoff[0] == 0 and np.all(np.diff(zoff) >= 0)
    assert zoff[-1] == rows * cpr
    assert chunk * ob <= (256 << 10) + 64 * ob
    per = np.diff(zoff)
    if cpr > 1:
        assert per.max() - per.min() <= max(2, per.max() // 4)
