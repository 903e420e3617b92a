"""LIBSVM ingestion against the reference's own outputs
(tests/golden/ingest.npz, written by oracle/make_golden.py from reference
data.py:31-254).  Host logic only: runs on CPU."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from conftest import golden  # noqa: E402
from paper_2410_08760_b200 import ingest  # noqa: E402

# the same crafted inputs the fixture generator parsed with the reference
GOOD = (
    b"# comment line\n"
    b"+1 1:0.5 3:2 7:-1.25e-3\n"
    b"\n"
    b"-1\t2:1 3:1\r\n"
    b"  +1 4:3.0000000000000004   9:1e300\n"
    b"-1 1:-0 2:0.1\n"
    b"+1\n"
    b"-1 5:7 6:8 8:9\n"
    b"+1 1:1 2:2 3:3 4:4\n"
    b"   # indented comment\n"
    b"-1 9:0.3333333333333333\n"
)
BAD = {
    "bad_label": b"+1 1:1\nabc 2:3\n",
    "three_labels": b"1 1:1\n2 1:1\n3 1:1\n",
    "no_colon": b"1 1:1\n0 2 3:1\n",
    "bad_index": b"1 x:1\n",
    "index_zero": b"1 0:1\n",
    "not_increasing": b"1 3:1 3:2\n",
    "decreasing": b"1   5:1   2:2\n",
    "bad_value": b"1 1:1 2:abc\n",
    "empty": b"# only\n\n",
}


def _rows(lens, idx, val):
    out, o = [], 0
    for n in lens:
        out.append((idx[o:o + n].astype(np.int64), val[o:o + n]))
        o += n
    return out


def test_parse_and_write_match_reference():
    g = golden("ingest.npz")
    ds = ingest.parse_libsvm(GOOD)
    assert np.array_equal(ds.labels, g["good__labels"])
    assert ds.num_features == int(g["good__num_features"])
    assert [len(r[0]) for r in ds.rows] == g["good__lens"].tolist()
    assert np.array_equal(np.concatenate([r[0] for r in ds.rows]), g["good__idx"])
    got_val = np.concatenate([r[1] for r in ds.rows])
    assert np.array_equal(got_val.view(np.uint64), g["good__val"].view(np.uint64))  # -0.0 kept
    written = ingest.write_libsvm(ds)
    assert written == g["good__written"].tobytes()
    again = ingest.parse_libsvm(written)
    assert np.array_equal(again.labels, ds.labels)
    assert all(np.array_equal(a[1], b[1]) for a, b in zip(again.rows, ds.rows))


@pytest.mark.parametrize("name", list(BAD))
def test_parse_errors_match_reference_positions(name):
    g = golden("ingest.npz")
    with pytest.raises(ingest.ParseError) as e:
        ingest.parse_libsvm(BAD[name])
    assert [e.value.line, e.value.col] == g[f"bad_{name}"].tolist()
    assert str(e.value) == str(g[f"bad_{name}__msg"])


def test_normalize_labels_conventions():
    g = golden("ingest.npz")
    for lo, hi in ((0.0, 1.0), (-1.0, 1.0), (2.0, 7.0)):
        raw = ingest.RawDataset(labels=np.array([hi, lo, hi]), rows=[(np.zeros(0, np.int64), np.zeros(0))] * 3,
                                num_features=1)
        ingest.normalize_labels(raw)
        assert np.array_equal(raw.labels, g[f"norm_{lo:g}_{hi:g}"])
    with pytest.raises(ValueError):
        ingest.normalize_labels(ingest.RawDataset(labels=np.array([1.0, 1.0]), rows=[], num_features=0))


def test_augment_and_shard_bytes_match_reference():
    g = golden("ingest.npz")
    ds = ingest.RawDataset(labels=g["shard__labels"].copy(),
                           rows=_rows(g["shard__lens"], g["shard__idx"], g["shard__val"]), num_features=11)
    shards = ingest.augment_and_shard(ds, 4, 9, 0.01)
    want = g["shard__bmats"]
    assert len(shards) == 4
    for s, w in zip(shards, want):
        assert s.bmat.flags.f_contiguous and s.lam == 0.01
        assert np.array_equal(s.bmat, w)
    pieces = ingest.split_rows(ds, 4, 9)
    assert np.array_equal(np.stack([p.labels for p in pieces]), g["shard__split_labels"])
    with pytest.raises(ValueError):  # labels not yet normalized
        ingest.augment_and_shard(ingest.RawDataset(np.array([0.0, 1.0]), ds.rows[:2], 11), 1, 0, 0.1)
    with pytest.raises(ValueError):  # more clients than samples
        ingest.augment_and_shard(ds, 24, 9, 0.01)


def test_load_client_shard_pads_features(tmp_path):
    p = tmp_path / "c0.libsvm"
    p.write_bytes(b"0 1:2 3:4\n1 2:5\n")
    s = ingest.load_client_shard(str(p), lam=0.5, num_features=5)
    assert s.bmat.shape == (6, 2)
    assert np.array_equal(s.bmat[:, 0], [-2.0, 0.0, -4.0, 0.0, 0.0, -1.0])
    assert np.array_equal(s.bmat[:, 1], [0.0, 5.0, 0.0, 0.0, 0.0, 1.0])
    with pytest.raises(ValueError):
        ingest.load_client_shard(str(p), lam=0.5, num_features=2)
