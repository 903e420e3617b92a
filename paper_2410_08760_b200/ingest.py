"""LIBSVM ingestion into client shards (host side, one-time, untimed).

Mirrors the reference's data pipeline for real datasets (
reference data.py:31-245): `parse_libsvm` / `load_libsvm` (1-based sparse
rows, two label values, `ParseError` with 1-based line and column),
`write_libsvm` (round-trips exactly, %.17g), `normalize_labels` ({0,1} and
other pairs onto {-1,+1}), `augment_and_shard` (TAG_SHUFFLE Fisher-Yates,
equal shards of floor(m/n) rows, intercept last, label absorbed),
`split_rows` and `load_client_shard`.  The dense shards it returns are what
`simulate` uploads to the device.

The parser walks each line's whitespace-separated tokens with their byte
offsets (so the reported column is the token's first byte, as the
reference reports it) and accepts exactly the token syntax Python's
int() / float() accept, as the reference does.
"""

from __future__ import annotations

import logging
import re
from dataclasses import dataclass

import numpy as np

from .data import ClientShard, shard_permutation

log = logging.getLogger(__name__)

_TOKEN = re.compile(rb"\S+")


class ParseError(Exception):
    """Malformed LIBSVM input (data.py:31-38): 1-based line and column."""

    def __init__(self, line: int, col: int, reason: str):
        self.line = line
        self.col = col
        super().__init__(f"line {line}, column {col}: {reason}")


@dataclass
class RawDataset:
    """Labels plus sparse rows with 1-based feature indices (data.py:41-50)."""

    labels: np.ndarray
    rows: list[tuple[np.ndarray, np.ndarray]]
    num_features: int

    @property
    def n_samples(self) -> int:
        return len(self.rows)


def _parse_row(line: bytes, lineno: int, toks: list) -> tuple[np.ndarray, np.ndarray, int]:
    idx = np.empty(len(toks), dtype=np.int64)
    val = np.empty(len(toks))
    last = 0
    for n, m in enumerate(toks):
        tok, col = m.group(0), m.start() + 1
        colon = tok.find(b":")
        if colon < 0:
            raise ParseError(lineno, col, f"feature {tok!r} lacks ':'")
        head, tail = tok[:colon], tok[colon + 1:]
        try:
            i = int(head)
        except ValueError:
            raise ParseError(lineno, col, f"bad feature index {head!r}") from None
        if i < 1:
            raise ParseError(lineno, col, f"feature index {i} < 1")
        if i <= last:
            raise ParseError(lineno, col, f"feature index {i} not increasing")
        try:
            x = float(tail)
        except ValueError:
            raise ParseError(lineno, col, f"bad feature value {tail!r}") from None
        idx[n], val[n], last = i, x, i
    return idx, val, last


def parse_libsvm(buf: bytes | bytearray | memoryview) -> RawDataset:
    """LIBSVM bytes -> RawDataset; blank and '#' lines are skipped."""
    labels: list[float] = []
    rows: list[tuple[np.ndarray, np.ndarray]] = []
    seen: set[float] = set()
    width = 0
    for lineno, line in enumerate(bytes(buf).split(b"\n"), start=1):
        toks = list(_TOKEN.finditer(line))
        if not toks or toks[0].group(0).startswith(b"#"):
            continue
        head = toks[0]
        try:
            y = float(head.group(0))
        except ValueError:
            raise ParseError(lineno, head.start() + 1, f"bad label {head.group(0)!r}") from None
        seen.add(y)
        if len(seen) > 2:
            raise ParseError(lineno, head.start() + 1, "more than two distinct labels")
        idx, val, last = _parse_row(line, lineno, toks[1:])
        width = max(width, last)
        labels.append(y)
        rows.append((idx, val))
    if not rows:
        raise ParseError(1, 1, "dataset is empty")
    return RawDataset(labels=np.array(labels), rows=rows, num_features=width)


def load_libsvm(path: str) -> RawDataset:
    with open(path, "rb") as fh:
        return parse_libsvm(fh.read())


def write_libsvm(ds: RawDataset) -> bytes:
    """Bytes that parse back to an identical dataset (data.py:116-126)."""
    lines = []
    for y, (idx, val) in zip(ds.labels, ds.rows):
        lines.append(b" ".join([b"%.17g" % y] + [b"%d:%.17g" % (int(i), x) for i, x in zip(idx, val)]))
    return b"\n".join(lines) + b"\n"


def normalize_labels(ds: RawDataset) -> None:
    """Two label values onto {-1, +1} in place (data.py:129-144): {-1, +1}
    kept, {0, 1} maps 0 to -1, any other pair maps the smaller to -1."""
    vals = sorted(set(ds.labels.tolist()))
    if len(vals) == 1:
        raise ValueError(f"dataset has a single label value {vals[0]!r}")
    lo, hi = vals
    if (lo, hi) == (-1.0, 1.0):
        return
    if (lo, hi) != (0.0, 1.0):
        log.info("labels {%g, %g}: mapping %g -> -1, %g -> +1", lo, hi, lo, hi)
    ds.labels = np.where(ds.labels == lo, -1.0, 1.0)


def _dense_columns(ds: RawDataset, sel: np.ndarray, d: int) -> np.ndarray:
    """Columns label * (features, 1) of the rows `sel`, F-order d x len(sel)."""
    b = np.zeros((d, len(sel)), order="F")
    for col, r in enumerate(sel):
        idx, val = ds.rows[r]
        if len(idx):
            b[idx - 1, col] = val
    b[d - 1, :] = 1.0
    b *= ds.labels[sel]
    return b


def augment_and_shard(ds: RawDataset, n_clients: int, run_seed: int, lam: float) -> list[ClientShard]:
    """Shuffle (TAG_SHUFFLE), equal shards, intercept last, labels absorbed
    (data.py:186-213).  Labels must already be in {-1, +1}."""
    seen = set(np.unique(ds.labels).tolist())
    if not seen <= {-1.0, 1.0}:
        raise ValueError(f"labels must be normalized to -1/+1, got {sorted(seen)}")
    perm, per = shard_permutation(ds.n_samples, n_clients, run_seed)
    dropped = ds.n_samples - per * n_clients
    if dropped:
        log.info("dropping %d of %d samples to equalize %d shards", dropped, ds.n_samples, n_clients)
    d = ds.num_features + 1
    return [ClientShard(bmat=_dense_columns(ds, perm[c * per:(c + 1) * per], d), lam=lam)
            for c in range(n_clients)]


def split_rows(ds: RawDataset, n_clients: int, run_seed: int) -> list[RawDataset]:
    """Per-client raw pieces with the same shuffle and slicing (data.py:216-233)."""
    perm, per = shard_permutation(ds.n_samples, n_clients, run_seed)
    out = []
    for c in range(n_clients):
        sel = perm[c * per:(c + 1) * per]
        out.append(RawDataset(labels=ds.labels[sel].copy(), rows=[ds.rows[i] for i in sel],
                              num_features=ds.num_features))
    return out


def load_client_shard(path: str, lam: float, num_features: int | None = None) -> ClientShard:
    """One client's LIBSVM file as a dense shard, no shuffle (data.py:236-254);
    `num_features` pads the dimension to the global feature count."""
    ds = load_libsvm(path)
    normalize_labels(ds)
    if num_features is not None:
        if num_features < ds.num_features:
            raise ValueError(f"--features {num_features} below max index {ds.num_features}")
        ds.num_features = num_features
    return ClientShard(bmat=_dense_columns(ds, np.arange(ds.n_samples), ds.num_features + 1), lam=lam)
