"""prune_stage (pruning.py:262-335) against patterns the
REAL reference produced (tests/golden/make_golden_prune.py): magnitude,
heterogeneous and tied scores, G = 16/32/64/128 with remainder tiles, and
two-stage runs (prev).  CPU: the host selection logic with the reductions
emulated in the kernels' summation order (and that order checked against
numpy's own means, bit for bit).  GPU: the whole stage with the CUDA score
kernels."""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2008_13006_b200 as tw
from paper_2008_13006_b200 import pruning

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_prune.npz"))


def cases():
    for i in range(int(GOLD["n_cases"])):
        c = {key[len(f"c{i}_"):]: GOLD[key] for key in GOLD.files if key.startswith(f"c{i}_")}
        w = c["w"]
        s = np.abs(w.astype(np.float64))
        if int(c["ties"]):
            s = np.round(s * 2) / 2
        c["s"] = s
        yield i, c


def pattern_of(c, tag, k, n, g):
    if f"{tag}_cols" not in c:
        return None
    cols, off, keep = c[f"{tag}_cols"], c[f"{tag}_off"], c[f"{tag}_keep"]
    return tw.TilePattern(k, n, g, tuple(tw.Tile(cols[off[t]:off[t + 1]], keep[t]) for t in range(off.size - 1)))


def same(p, q):
    return (len(p.tiles) == len(q.tiles) and
            all(np.array_equal(a.col_ids, b.col_ids) and np.array_equal(a.row_keep, b.row_keep)
                for a, b in zip(p.tiles, q.tiles)))


class SeqMeans:
    """The CUDA kernels' order on the host: sequential float64 sums."""

    def __init__(self, s):
        self.s = s

    def cols(self):
        acc = np.zeros(self.s.shape[1])
        for r in range(self.s.shape[0]):
            acc += self.s[r]
        return acc / self.s.shape[0]

    def rows(self, cols, off):
        out = []
        for t in range(off.size - 1):
            sub = self.s[:, cols[off[t]:off[t + 1]]]
            acc = np.zeros(self.s.shape[0])
            for j in range(sub.shape[1]):
                acc += sub[:, j]
            out.append(acc / sub.shape[1])
        return np.concatenate(out)


@pytest.mark.parametrize("i,c", list(cases()))
def test_prune_stage_host_logic_matches_reference(i, c):
    k, n, g, s_t = int(c["k"]), int(c["n"]), int(c["g"]), float(c["s_t"])
    s = c["s"]
    # the kernels' summation order IS numpy's (pruning.py:293, :316)
    sm = SeqMeans(s)
    assert np.array_equal(sm.cols(), s.mean(axis=0))
    prev = None
    if int(c["staged"]):
        prev = pruning.prune_stage(c["w"], s, float(c["prev_s_t"]), g, _means=SeqMeans)
        assert same(prev, pattern_of(c, "prev", k, n, g))
    got = pruning.prune_stage(c["w"], s, s_t, g, prev=prev, _means=SeqMeans)
    assert same(got, pattern_of(c, "out", k, n, g))


def test_select_units_contract():
    s = np.array([3.0, 1.0, 1.0, 0.5, 2.0])
    assert list(pruning.select_units(s, 2, [], [])) == [1, 3]          # ties by index
    assert list(pruning.select_units(s, 2, [4], [])) == [3, 4]         # forced first
    assert list(pruning.select_units(s, 2, [], [3])) == [1, 2]         # protected skipped
    with pytest.raises(tw.ConfigError):
        pruning.select_units(s, 5, [], [0])
    with pytest.raises(tw.ConfigError):
        pruning.prune_stage(np.zeros((4, 4), np.float32), np.zeros((4, 4)), 1.0, 2, _means=SeqMeans)


@pytest.mark.gpu
@pytest.mark.parametrize("i,c", list(cases()))
def test_prune_stage_gpu_matches_reference(i, c):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    k, n, g, s_t = int(c["k"]), int(c["n"]), int(c["g"]), float(c["s_t"])
    s = c["s"]
    gm = pruning._GpuMeans(s, None)
    assert np.array_equal(gm.cols(), s.mean(axis=0))  # bit-identical float64 means
    prev = None
    if int(c["staged"]):
        prev = tw.prune_stage(c["w"], s, float(c["prev_s_t"]), g)
        assert same(prev, pattern_of(c, "prev", k, n, g))
    assert same(tw.prune_stage(c["w"], s, s_t, g, prev=prev), pattern_of(c, "out", k, n, g))
