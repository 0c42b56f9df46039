"""GPU parity of K4, the CTA-pair kernel (tcgen05 cta_group::2) that runs
plans whose tiles keep every K row: dense patterns (gemm_dense, BERT-large
at 0 %) and TW_PLAN_DENSE_PAD plans of near-dense patterns (pruned weights
as zeros).  Same bar as every tensor-core path: rel-L2 <= 1e-3 against the
CPU oracle (the reference's fp32 algorithm, engine.py:152-164) on the same
bf16-rounded inputs, pruned output columns exactly 0.  Each test also checks
from the profiler's kernel list that K4 (or, for dense_pad=False, K2) ran.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2008_13006_b200 as tw  # noqa: E402
from oracle import oracle as orc  # noqa: E402

pytestmark = pytest.mark.gpu
RTOL = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert torch.cuda.get_device_capability()[0] == 10, "sm_100 (B200) required"


def kernels_of(fn):
    """Names of the CUDA kernels fn() launches (torch profiler)."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = fn()
        torch.cuda.synchronize()
    return r, {e.name for e in prof.events() if e.device_type.name == "CUDA"}


def run_case(m, k, n, g, s, seed=3, out_dtype=torch.float32, dense_pad=None, pattern=None, bias=None, relu=False):
    a, w, p = orc.bench_inputs(m, k, n, g, s, seed=seed)
    if pattern is not None:
        p = pattern
    pat = tw.TilePattern(p[0], p[1], p[2], tuple(tw.Tile(c, keep) for c, keep in p[3])) \
        if isinstance(p, tuple) else p
    ts = tw.compact(tw.DenseMatrix.from_array(w), pat)
    plan = tw.TwPlan(ts, dense_pad=dense_pad)
    at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    bias_t = torch.from_numpy(bias).cuda() if bias is not None else None
    ct, names = kernels_of(lambda: plan.gemm(at, out_dtype=out_dtype, bias=bias_t, relu=relu)
                           if bias is not None else plan.gemm(at, out_dtype=out_dtype))
    sub = orc.compact(w, p)
    want = orc.gemm_tw_ct(np.ascontiguousarray(a.T), orc.PackedTiles(sub, k, n), threads=orc.max_threads())
    if bias is not None:
        want = want + bias[:, None]
        if relu:
            want = np.maximum(want, 0)
    return plan, ct.float().cpu().numpy(), want, orc.pruned_columns(p), names


def ran_pair(names):
    return any("tw_pair_sm100_kernel" in x for x in names)


@pytest.mark.parametrize("m,k,n", [(512, 256, 512), (1024, 768, 768), (320, 192, 256), (4096, 1024, 1024)])
def test_dense_pattern_runs_on_pair_kernel(m, k, n):
    plan, ct, want, _, names = run_case(m, k, n, 128, 0.0, dense_pad=True)
    assert ran_pair(names), names
    assert rel_l2(ct, want) < 1e-5


def rel_l2(got, want):
    return orc.rel_l2(got, want)


@pytest.mark.parametrize("out_dtype,bar", [(torch.float32, 1e-5), (torch.float16, 1e-3), (torch.bfloat16, 5e-3)])
def test_dense_pad_plan_vs_oracle(out_dtype, bar):
    # a 40 %-sparse TW pattern packed dense: pruned rows are zero weights,
    # pruned columns stay exactly zero
    plan, ct, want, prc, names = run_case(2048, 768, 1536, 128, 0.4, out_dtype=out_dtype, dense_pad=True)
    assert plan.dense_padded and ran_pair(names), names
    assert np.all(ct[prc] == 0.0)
    assert rel_l2(ct, want) <= bar, rel_l2(ct, want)


def test_dense_layer_at_full_wave_runs_k4_by_default():
    # no dense_pad argument: a dense 4096 x 1024 x 4096 layer fills the CTA pairs
    plan, ct, want, _, names = run_case(4096, 1024, 4096, 128, 0.0)
    assert plan.kernel_for(4096) == 4 and ran_pair(names), names
    assert rel_l2(ct, want) < 1e-5


def test_dense_pad_off_keeps_gather_kernel():
    plan, ct, want, prc, names = run_case(1024, 512, 1024, 128, 0.2, dense_pad=False)
    assert not plan.dense_padded and not ran_pair(names), names
    assert rel_l2(ct, want) < 1e-5


def test_auto_choice_follows_density():
    _, w, p_dense = orc.bench_inputs(8, 256, 512, 128, 0.1, seed=1)
    _, _, p_sparse = orc.bench_inputs(8, 256, 512, 128, 0.75, seed=1)
    to = lambda p: tw.TilePattern(p[0], p[1], p[2], tuple(tw.Tile(c, keep) for c, keep in p[3]))  # noqa: E731
    assert tw.TwPlan(tw.compact(tw.DenseMatrix.from_array(w), to(p_dense))).dense_padded
    assert not tw.TwPlan(tw.compact(tw.DenseMatrix.from_array(w), to(p_sparse))).dense_padded


@pytest.mark.parametrize("n", [128, 384, 640])
def test_odd_tile_count(n):
    # the last CTA pair has one tile: the follower computes a copy and stores nothing
    plan, ct, want, _, names = run_case(768, 256, n, 128, 0.0, dense_pad=True)
    assert ran_pair(names)
    assert rel_l2(ct, want) < 1e-5


@pytest.mark.parametrize("m", [16, 136, 1000, 2056])
def test_ragged_m(m):
    # tokens past M: zero-filled by the TMA loads, clipped by the TMA stores
    plan, ct, want, _, names = run_case(m, 384, 512, 128, 0.0, dense_pad=True)
    assert ran_pair(names)
    assert ct.shape == (512, m)
    assert rel_l2(ct, want) < 1e-5


def test_non_consecutive_tile_columns_and_dead_tiles():
    # tiles over scattered columns (bulk row stores instead of TMA tensor
    # stores) and a fully pruned tile (zero rows)
    k, n, g = 256, 640, 128
    rng = np.random.default_rng(5)
    perm = rng.permutation(n)
    tiles = []
    for t in range(5):
        cols = np.sort(perm[t * 128:(t + 1) * 128]).astype(np.int32)
        keep = np.ones(k, dtype=bool)
        if t == 3:
            keep[:] = False  # dead tile: its columns are zero rows of C^T
        elif t == 1:
            keep[rng.choice(k, 40, replace=False)] = False
        tiles.append((cols, keep))
    plan, ct, want, prc, names = run_case(512, k, n, g, 0.0, pattern=(k, n, g, tiles), dense_pad=True)
    assert ran_pair(names)
    assert np.all(ct[tiles[3][0]] == 0.0)  # the dead tile's columns
    assert rel_l2(ct, want) < 1e-5


@pytest.mark.parametrize("relu,out_dtype", [(True, torch.float16), (False, torch.float32)])
def test_bias_relu_epilogue(relu, out_dtype):
    n = 512
    bias = np.random.default_rng(2).standard_normal(n).astype(np.float32)
    plan, ct, want, _, names = run_case(1024, 512, n, 128, 0.0, out_dtype=out_dtype, bias=bias, relu=relu,
                                        dense_pad=True)
    assert ran_pair(names)
    assert rel_l2(ct, want) <= (1e-3 if out_dtype == torch.float16 else 1e-5)


def test_pair_and_gather_kernels_agree():
    # the same near-dense layer through K4 (dense-padded) and K2 (kept rows)
    a, w, p = orc.bench_inputs(1536, 512, 1024, 128, 0.3, seed=9)
    pat = tw.TilePattern(p[0], p[1], p[2], tuple(tw.Tile(c, keep) for c, keep in p[3]))
    ts = tw.compact(tw.DenseMatrix.from_array(w), pat)
    at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    c4 = tw.TwPlan(ts, dense_pad=True).gemm(at).cpu().numpy()
    c2 = tw.TwPlan(ts, dense_pad=False).gemm(at).cpu().numpy()
    assert rel_l2(c4, c2) < 1e-6


def test_back_to_back_launches_and_graph_replay():
    # PDL-chained launches and a captured graph over rotating outputs
    a, w, p = orc.bench_inputs(2048, 512, 1024, 128, 0.0, seed=4)
    pat = tw.TilePattern(p[0], p[1], p[2], tuple(tw.Tile(c, keep) for c, keep in p[3]))
    plan = tw.TwPlan(tw.compact(tw.DenseMatrix.from_array(w), pat), dense_pad=True)
    at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    ref, names = kernels_of(lambda: plan.gemm(at, out_dtype=torch.float16))
    assert ran_pair(names)
    outs = [torch.empty_like(ref) for _ in range(4)]
    for i in range(20):
        plan.gemm(at, out=outs[i % 4], out_dtype=torch.float16)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(8):
            plan.gemm(at, out=outs[i % 4], out_dtype=torch.float16)
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)


def test_small_auto_padded_layer_launches_unpadded_plan_on_k2():
    # C1 (1024^3 @ 50 %, 71 % of rows kept) is auto-padded, but its 12 pair
    # units fill 12 of 74 CTA pairs: gemm() runs the unpadded sibling on K2
    plan, ct, want, prc, names = run_case(1024, 1024, 1024, 128, 0.5)
    assert plan.dense_padded
    assert plan.kernel_for(1024) == 2 and not ran_pair(names), names
    assert np.all(ct[prc] == 0.0)
    assert rel_l2(ct, want) < 1e-5
    # the same plan at a large M fills the pairs
    assert plan.kernel_for(16384) == 4


def test_column_range_shard_of_a_padded_plan():
    # the N-sharded unit: a shard [c0, c1) cuts tiles (n_i < 128, scattered
    # rows) -- K4 stores them through the LSU path; rows re-based to 0
    a, w, p = orc.bench_inputs(2048, 512, 1024, 128, 0.3, seed=11)
    pat = tw.TilePattern(p[0], p[1], p[2], tuple(tw.Tile(c, keep) for c, keep in p[3]))
    ts = tw.compact(tw.DenseMatrix.from_array(w), pat)
    at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    want = orc.gemm_tw_ct(np.ascontiguousarray(a.T), orc.PackedTiles(orc.compact(w, p), 512, 1024),
                          threads=orc.max_threads())
    for c0, c1 in ((0, 512), (100, 900), (777, 1024)):
        plan = tw.TwPlan(ts, col_range=(c0, c1), dense_pad=True)
        ct, names = kernels_of(lambda: plan.gemm(at, out_dtype=torch.float16))
        assert ran_pair(names)
        assert rel_l2(ct.float().cpu().numpy(), want[c0:c1]) <= 1e-3


def test_resident_output_keep_pruned():
    # write_pruned=False: the pruned rows of a reused buffer keep their value
    plan, ct, want, prc, names = run_case(2048, 512, 1024, 128, 0.3, dense_pad=True)
    a, w, p = orc.bench_inputs(2048, 512, 1024, 128, 0.3, seed=3)
    at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    out = torch.full((1024, 2048), 7.0, dtype=torch.float32, device="cuda")
    plan.gemm(at, out=out, write_pruned=False)
    got = out.cpu().numpy()
    kept = np.setdiff1d(np.arange(1024), prc)
    assert np.all(got[prc] == 7.0)
    assert rel_l2(got[kept], want[kept]) < 1e-5


def test_fp16_operands():
    a, w, p = orc.bench_inputs(1024, 512, 1024, 128, 0.1, seed=5)
    pat = tw.TilePattern(p[0], p[1], p[2], tuple(tw.Tile(c, keep) for c, keep in p[3]))
    ts = tw.compact(tw.DenseMatrix.from_array(w), pat)
    plan = tw.TwPlan(ts, dtype=torch.float16, dense_pad=True)
    at = tw.prep_activations(torch.from_numpy(a).cuda(), tw.Layout.ROW_MAJOR, torch.float16)
    ct, names = kernels_of(lambda: plan.gemm(at))
    assert ran_pair(names)
    want = orc.gemm_tw_ct(np.ascontiguousarray(a.T), orc.PackedTiles(orc.compact(w, p), 512, 1024),
                          threads=orc.max_threads())
    # fp16 operands round A and W differently from the bf16-rounded oracle inputs
    assert rel_l2(ct.cpu().numpy(), want) <= 1e-3


def test_layer_chain_through_near_dense_layers():
    # TwMlp with near-dense layers (auto-padded, K4 at this size) feeding each
    # layer's C^T in as the next A^T, against the oracle layer by layer
    rng = np.random.default_rng(8)
    m, dims = 8192, [512, 1024, 512]
    pats, ws, bs = [], [], []
    for i in range(2):
        k, n = dims[i], dims[i + 1]
        _, w, p = orc.bench_inputs(8, k, n, 128, 0.15, seed=20 + i)
        pats.append(p)
        ws.append(w)
        bs.append(rng.standard_normal(n).astype(np.float32))
    layers = []
    for p, w, b in zip(pats, ws, bs):
        pat = tw.TilePattern(p[0], p[1], p[2], tuple(tw.Tile(c, keep) for c, keep in p[3]))
        plan = tw.TwPlan(tw.compact(tw.DenseMatrix.from_array(w), pat))
        assert plan.dense_padded
        layers.append((plan, torch.from_numpy(b).cuda()))
    x = orc.bf16_round(rng.standard_normal((m, dims[0])).astype(np.float32))
    at = tw.prep_activations(torch.from_numpy(x).cuda(), tw.Layout.ROW_MAJOR, torch.bfloat16)
    ref = np.ascontiguousarray(x.T)
    for li, ((plan, b), p, w) in enumerate(zip(layers, pats, ws)):
        last = li == len(layers) - 1
        ct, names = kernels_of(lambda: plan.gemm(at, out_dtype=torch.float32 if last else torch.bfloat16,
                                                 bias=b, relu=not last))
        assert ran_pair(names)
        want = orc.gemm_tw_ct(ref, orc.PackedTiles(orc.compact(w, p), w.shape[0], w.shape[1]),
                              threads=orc.max_threads()) + bs[li][:, None]
        if not last:
            want = np.maximum(want, 0)
        got = ct.float().cpu().numpy()
        assert rel_l2(got, want) <= (5e-3 if not last else 1e-3), (li, rel_l2(got, want))
        at = ct  # C^T of this layer is A^T of the next
        ref = got.astype(np.float32)  # the oracle continues from the GPU's rounded activations
