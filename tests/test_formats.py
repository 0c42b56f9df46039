"""TWPT / TWCS / TWMX readers and writers against
files written by the reference itself (tests/golden/make_golden_formats.py),
and the file -> packer path (formats.plan_from_files) against the packer fed
from compact().  CPU only."""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2008_13006_b200 as tw
from paper_2008_13006_b200 import formats

FMT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fmt")


def f(name):
    return os.path.join(FMT, name)


@pytest.mark.parametrize("name", ["c2b.twpt", "g64.twpt"])
def test_pattern_roundtrip_byte_identical(name, tmp_path):
    p = tw.read_pattern(f(name))
    out = tmp_path / name
    tw.write_pattern(p, out)
    assert open(out, "rb").read() == open(f(name), "rb").read()


def test_pattern_contents():
    p = tw.read_pattern(f("c2b.twpt"))
    assert (p.k, p.n, p.g) == (768, 768, 128)
    assert len(p.tiles) == 3 and all(t.n_i == 128 and t.k_i == 384 for t in p.tiles)


def test_matrix_and_csc_roundtrip(tmp_path):
    for name in ("w_g64.twmx", "w_g64_col.twmx"):
        m = tw.read_matrix(f(name))
        assert (m.rows, m.cols) == (96, 150)
        tw.write_matrix(m, tmp_path / name)
        assert open(tmp_path / name, "rb").read() == open(f(name), "rb").read()
    a, b = tw.read_matrix(f("w_g64.twmx")), tw.read_matrix(f("w_g64_col.twmx"))
    assert np.array_equal(a.array(), b.array())
    s = tw.read_csc(f("ew_g64.twcs"))
    assert s.rows == 96 and s.cols == 150 and s.nnz > 0
    tw.write_csc(s, tmp_path / "x.twcs")
    assert open(tmp_path / "x.twcs", "rb").read() == open(f("ew_g64.twcs"), "rb").read()


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "bad magic"),
    (lambda b: b[:10], "truncated"),
    (lambda b: b + b"\0", "trailing"),
    (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "version"),
])
def test_corrupt_files_raise_format_error(mutate, msg, tmp_path):
    for name, reader in (("g64.twpt", tw.read_pattern), ("w_g64.twmx", tw.read_matrix),
                         ("ew_g64.twcs", tw.read_csc)):
        raw = open(f(name), "rb").read()
        path = tmp_path / ("bad_" + name)
        path.write_bytes(mutate(raw))
        with pytest.raises(tw.FormatError):
            reader(path)


def test_plan_from_files_matches_compact_path():
    ref = tw.PackedPlan(tw.compact(tw.read_matrix(f("w_g64.twmx")), tw.read_pattern(f("g64.twpt"))))
    for wname in ("w_g64.twmx", "w_g64_col.twmx"):
        got = formats.plan_from_files(f("g64.twpt"), f(wname), host=True)
        for which in ("kidx", "colids", "zero_rows", "wimg", "tiles"):
            assert np.array_equal(got.export(which), ref.export(which)), which
        assert got.info == ref.info


def test_plan_from_files_dimension_mismatch():
    with pytest.raises(tw.DimensionError):
        formats.plan_from_files(f("c2b.twpt"), f("w_g64.twmx"), host=True)


def test_read_model_reference_checkpoint(tmp_path):
    ws, bs = tw.read_model(f("mlp.twml"))
    assert [w.shape for w in ws] == [(64, 96), (96, 10)] and [b.shape for b in bs] == [(96,), (10,)]
    raw = open(f("mlp.twml"), "rb").read()
    for i, bad in enumerate((raw[:30], raw + b"\0", b"XXXX" + raw[4:])):
        p = tmp_path / f"bad{i}.twml"
        p.write_bytes(bad)
        with pytest.raises(tw.FormatError):
            tw.read_model(p)


def test_cli_exit_codes_without_gpu(tmp_path, capsys):
    from paper_2008_13006_b200 import cli
    # config error (repeats < 5, cli.py:383-384) -> 2
    assert cli.main(["bench", "--repeats", "3", "--out", str(tmp_path / "b.csv")]) == cli.EXIT_CONFIG
    # missing pattern files -> I/O error 3
    assert cli.main(["verify", "--model", f("mlp.twml"), "--patterns", str(tmp_path)]) == cli.EXIT_IO
    # malformed checkpoint -> format error 3
    bad = tmp_path / "bad.twml"
    bad.write_bytes(b"TWMLxx")
    assert cli.main(["verify", "--model", str(bad), "--patterns", FMT]) == cli.EXIT_IO
