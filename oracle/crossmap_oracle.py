"""CPU oracle for the cross-map hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``crossmap`` package's
hot path (``/root/reference/pkg/src/crossmap``).  It exists to CHECK the
B200 path, never to BE it: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.
The product package (``paper_2105_12301_b200``) never imports this file and
raises when its CUDA library is missing.

Parity pinning: ``tests/test_oracle.py`` checks every function here against
(a) the known-answer vectors frozen in the reference's own tests
(pkg/tests/test_knn.py:19-22, test_prediction.py:23-33) and (b) outputs of the
reference itself, generated in the build container by
``tests/golden/make_golden.py`` and committed as ``tests/golden/*.npz``.

Arithmetic follows the reference bit-for-bit where the reference is
deterministic: float64 values, squared distances accumulated coordinate by
coordinate in order e = 0..E-1 (knn.py:118-125), selection by the
lexicographic key (distance, index) with the query point excluded
(knn.py:164-172), weights exp(-d/dmin) with the degenerate-scale rules
(knn.py:194-202), block-wise two-pass Pearson aggregates merged with the
pooled-moment rule (prediction.py:45-79).

The one component with no reference implementation -- the library-size
convergence sweep ``ccm_convergence`` -- is
a restatement of the CCM literature's definition on top of the same
primitives; its parity is UNPINNED (no reference code or test exists,
SPEC.md:322, 331).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from math import sqrt

import numpy as np

#: knn.py:27 -- floor applied to exp() weights so they stay strictly positive.
TINY = np.finfo(np.float64).tiny
#: prediction.py:22 -- Pearson aggregates are formed per 4096-point block.
BLOCK = 4096
#: _parallel.py:18 -- row tile of the CPU backend.
ROW_TILE = 256


class OracleError(ValueError):
    """Precondition failure inside the oracle (mirrors errors.py:4-21 kinds)."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


# --------------------------------------------------------------------------
# execution helper (restates _parallel.py:21-50: fixed tiles, any worker
# count gives identical results because tiles write disjoint slices)
# --------------------------------------------------------------------------

def _workers(workers):
    if workers is None:
        env = os.environ.get("CROSSMAP_WORKERS")
        workers = int(env) if env else (os.cpu_count() or 1)
    return max(1, int(workers))


def _tiled(total, fn, workers, tile=ROW_TILE):
    spans = [(s, min(s + tile, total)) for s in range(0, total, tile)]
    w = min(_workers(workers), len(spans))
    if w <= 1:
        for s, e in spans:
            fn(s, e)
        return
    with ThreadPoolExecutor(max_workers=w) as pool:
        list(pool.map(lambda se: fn(*se), spans))


# --------------------------------------------------------------------------
# geometry (series.py:58-98)
# --------------------------------------------------------------------------

def point_count(length: int, E: int, tau: int) -> int:
    """series.py:79-81: L - (E-1)*tau delay vectors (may be <= 0)."""
    return length - (E - 1) * tau


def valid_count(length: int, E: int, tau: int) -> int:
    """series.py:84-98: embedded points, requiring at least E + 2."""
    n = point_count(length, E, tau)
    if length < 1 or n < E + 2:
        raise OracleError("too_short", f"length {length} gives {n} points for E={E}, tau={tau}")
    return n


# --------------------------------------------------------------------------
# kNN tables (knn.py:97-217)
# --------------------------------------------------------------------------

def squared_distances(x, E: int, tau: int, workers=None) -> np.ndarray:
    """knn.py:97-128: D[i, j] = sum_{e<E} (x[i+e*tau] - x[j+e*tau])^2, float64,
    accumulated in coordinate order (first term assigned, later ones added)."""
    x = np.asarray(x, dtype=np.float64)
    n = point_count(x.size, E, tau)
    if n < 2:
        raise OracleError("too_short", f"{n} embedded points")
    D = np.empty((n, n))
    cols = [x[e * tau: e * tau + n] for e in range(E)]

    def rows(lo, hi):
        acc = D[lo:hi]
        scratch = np.empty_like(acc)
        for e in range(E):
            np.subtract(x[lo + e * tau: hi + e * tau][:, None], cols[e][None, :], out=scratch)
            np.multiply(scratch, scratch, out=scratch)
            if e == 0:
                acc[:] = scratch
            else:
                acc += scratch

    _tiled(n, rows, workers)
    return D


def select_k(D: np.ndarray, k: int, workers=None):
    """knn.py:144-177: per row the k smallest entries over j != i, ordered by
    the key (value, column).  Returns (values float64[n,k], columns int64[n,k]).

    Restated as: kth = k-th smallest value of the row (self poisoned to +inf);
    keep every column strictly below kth plus the lowest-index columns equal
    to kth until k are kept; order the kept set by (value, column).
    """
    D = np.asarray(D, dtype=np.float64)
    n = D.shape[0]
    if not 1 <= k <= n - 1:
        raise OracleError("param", f"neighbor count must lie in [1, {n - 1}], got {k}")
    out_d = np.empty((n, k))
    out_i = np.empty((n, k), dtype=np.int64)

    def rows(lo, hi):
        blk = D[lo:hi].copy()
        r = np.arange(hi - lo)
        blk[r, np.arange(lo, hi)] = np.inf
        kth = np.partition(blk, k - 1, axis=1)[:, k - 1]
        below = blk < kth[:, None]
        at = blk == kth[:, None]
        room = k - below.sum(axis=1)
        keep = below | (at & (np.cumsum(at, axis=1) <= room[:, None]))
        cols = np.nonzero(keep)[1].reshape(hi - lo, k)          # ascending column
        vals = np.take_along_axis(blk, cols, axis=1)
        order = np.argsort(vals, axis=1, kind="stable")           # ties keep low column
        out_i[lo:hi] = np.take_along_axis(cols, order, axis=1)
        out_d[lo:hi] = np.take_along_axis(vals, order, axis=1)

    _tiled(n, rows, workers)
    return out_d, out_i


def simplex_weights(top_sq: np.ndarray) -> np.ndarray:
    """knn.py:180-202: w = exp(-d/scale) normalised, d = sqrt(squared); scale is
    d[0], else the first positive d, else 1 (all-zero row -> uniform); raw
    weights are floored at TINY."""
    sq = np.asarray(top_sq, dtype=np.float64)
    d = np.sqrt(sq)
    scale = d[:, 0].copy()
    for r in np.flatnonzero(scale == 0.0):
        pos = d[r][d[r] > 0.0]
        scale[r] = pos[0] if pos.size else 1.0
    raw = np.maximum(np.exp(-d / scale[:, None]), TINY)
    return raw / raw.sum(axis=1, keepdims=True)


def knn_table(x, E: int, tau: int = 1, k: int | None = None, workers=None):
    """knn.py:205-217 (build_knn_table): (indices int64[n,k], weights f64[n,k])."""
    x = np.asarray(x, dtype=np.float64)
    valid_count(x.size, E, tau)
    k = E + 1 if k is None else k
    D = squared_distances(x, E, tau, workers)
    d, i = select_k(D, k, workers)
    return i, simplex_weights(d)


# --------------------------------------------------------------------------
# Pearson aggregates (prediction.py:25-103)
# --------------------------------------------------------------------------

def agg_from_arrays(a, b):
    """prediction.py:45-55: (count, mean_a, mean_b, m2_a, m2_b, comoment)."""
    n = a.size
    if n == 0:
        return (0, 0.0, 0.0, 0.0, 0.0, 0.0)
    ma = float(a.mean())
    mb = float(b.mean())
    da = a - ma
    db = b - mb
    return (int(n), ma, mb, float(da @ da), float(db @ db), float(da @ db))


def agg_merge(x, y):
    """prediction.py:57-73: pooled-moment merge."""
    if x[0] == 0:
        return y
    if y[0] == 0:
        return x
    n = x[0] + y[0]
    ga = y[1] - x[1]
    gb = y[2] - x[2]
    pooled = x[0] * y[0] / n
    return (n, x[1] + ga * y[0] / n, x[2] + gb * y[0] / n,
            x[3] + y[3] + ga * ga * pooled, x[4] + y[4] + gb * gb * pooled,
            x[5] + y[5] + ga * gb * pooled)


def agg_rho(agg):
    """prediction.py:75-79: None when count < 2 or either m2 <= 0, else clipped."""
    if agg[0] < 2 or agg[3] <= 0.0 or agg[4] <= 0.0:
        return None
    return float(np.clip(agg[5] / sqrt(agg[3] * agg[4]), -1.0, 1.0))


def pearson(a, b):
    """prediction.py:82-103 without the error raising: blockwise aggregates."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    agg = (0, 0.0, 0.0, 0.0, 0.0, 0.0)
    for s in range(0, a.size, BLOCK):
        agg = agg_merge(agg, agg_from_arrays(a[s:s + BLOCK], b[s:s + BLOCK]))
    return agg_rho(agg)


# --------------------------------------------------------------------------
# lookup (prediction.py:122-161)
# --------------------------------------------------------------------------

def lookup(indices, weights, E: int, tau: int, targets, want_predictions=False, workers=None):
    """prediction.py:122-161: per target, predictions sum_k w * y[idx + (E-1)tau]
    over 4096-point blocks, skill from merged block aggregates.
    Returns (rho list with None for undefined, predictions list or None)."""
    idx = np.asarray(indices)
    w = np.asarray(weights, dtype=np.float64)
    n = idx.shape[0]
    off = (E - 1) * tau
    shifted = idx + off
    targets = [np.ascontiguousarray(np.asarray(t, dtype=np.float64)) for t in targets]
    rhos = [None] * len(targets)
    preds = [None] * len(targets)

    def one(t):
        y = targets[t]
        if y.size < n + off:
            raise OracleError("param", f"target {t} has {y.size} samples; need {n + off}")
        obs = y[off: off + n]
        p_all = np.empty(n) if want_predictions else None
        agg = (0, 0.0, 0.0, 0.0, 0.0, 0.0)
        for s in range(0, n, BLOCK):
            e = min(s + BLOCK, n)
            p = np.einsum("ij,ij->i", w[s:e], y[shifted[s:e]])
            agg = agg_merge(agg, agg_from_arrays(obs[s:e], p))
            if p_all is not None:
                p_all[s:e] = p
        rhos[t] = agg_rho(agg)
        preds[t] = p_all

    _tiled(len(targets), lambda lo, hi: [one(t) for t in range(lo, hi)], workers, tile=1)
    return rhos, (preds if want_predictions else None)


# --------------------------------------------------------------------------
# simplex / edim (prediction.py:164-262)
# --------------------------------------------------------------------------

def simplex(x, E: int, tau: int = 1, Tp: int = 1, workers=None):
    """prediction.py:164-182: table on x[:L-Tp], lookup of x[Tp:] (None if undefined)."""
    x = np.asarray(x, dtype=np.float64)
    idx, w = knn_table(x[: x.size - Tp], E, tau, workers=workers)
    return lookup(idx, w, E, tau, [x[Tp:]], workers=workers)[0][0]


def skill_curve(x, E_max: int, tau: int = 1, Tp: int = 1, workers=None):
    """prediction.py:197-240: rho for E = 1..E_max from one incrementally grown
    distance matrix (bit-identical to one-shot tables, prediction.py:199-204).
    Entries are None where skill is undefined."""
    x = np.asarray(x, dtype=np.float64)
    lib = x[: x.size - Tp]
    tgt = x[Tp:]
    n1 = lib.size
    D = np.empty((n1, n1))

    def base(lo, hi):
        np.subtract(lib[lo:hi, None], lib[None, :], out=D[lo:hi])
        np.multiply(D[lo:hi], D[lo:hi], out=D[lo:hi])

    _tiled(n1, base, workers)
    curve = {}
    for E in range(1, E_max + 1):
        nE = n1 - (E - 1) * tau
        if E > 1:
            col = lib[(E - 1) * tau: (E - 1) * tau + nE]

            def grow(lo, hi, col=col, nE=nE):
                sq = np.subtract(col[lo:hi, None], col[None, :])
                np.multiply(sq, sq, out=sq)
                D[lo:hi, :nE] += sq

            _tiled(nE, grow, workers)
        d, i = select_k(D[:nE, :nE], E + 1, workers)
        curve[E] = lookup(i, simplex_weights(d), E, tau, [tgt], workers=workers)[0][0]
    return curve


def optimal_e(curve: dict) -> int:
    """prediction.py:257-261: argmax with strict '>' so ties go to the smaller E."""
    best = 1
    for E in range(2, max(curve) + 1):
        if curve[E] > curve[best]:
            best = E
    return best


def edim(x, E_max: int = 20, tau: int = 1, Tp: int = 1, workers=None):
    """prediction.py:243-262 (optimal_embedding) -> (e_star | None, curve).
    A constant series yields (None, {}) (ccm.py:116-120 marks it undefined)."""
    x = np.asarray(x, dtype=np.float64)
    if x.min() == x.max():
        return None, {}
    valid_count(x.size - Tp, E_max, tau)
    curve = skill_curve(x, E_max, tau, Tp, workers)
    if any(v is None for v in curve.values()):
        return None, curve
    return optimal_e(curve), curve


# --------------------------------------------------------------------------
# all-to-all cross map (ccm.py:94-151)
# --------------------------------------------------------------------------

def xmap(series, e_star, tau: int = 1, workers=None, libraries=None, targets=None):
    """ccm.py:123-149: rho[lib, tgt] with the library embedded at E*(tgt),
    contemporaneous (Tp = 0) lookup, NaN where undefined or where either
    series has no E* (None / 0).  ``libraries`` / ``targets`` restrict the
    computed rows / columns (CPU-baseline sampling); other cells stay NaN.
    Also returns the number of tables built."""
    X = [np.asarray(s, dtype=np.float64) for s in series]
    N = len(X)
    stars = [None if (e is None or int(e) <= 0) else int(e) for e in e_star]
    libs = range(N) if libraries is None else libraries
    tgt_set = set(range(N) if targets is None else targets)
    groups: dict[int, list[int]] = {}
    for t, e in enumerate(stars):
        if e is not None and t in tgt_set:
            groups.setdefault(e, []).append(t)
    rho = np.full((N, N), np.nan)
    tables = 0
    for lib in libs:
        if stars[lib] is None:
            continue
        for E in sorted(groups):
            idx, w = knn_table(X[lib], E, tau, workers=workers)
            tables += 1
            ids = groups[E]
            r, _ = lookup(idx, w, E, tau, [X[t] for t in ids], workers=workers)
            for t, v in zip(ids, r):
                if v is not None:
                    rho[lib, t] = v
    return rho, tables


def xmap_rows(series, e_star, libraries, tau: int = 1, workers=None):
    """The rows ``libraries`` of xmap (ccm.py:131-149 restricted to those
    libraries) as a [len(libraries), N] array, without the N x N matrix (the
    sampled checks at N = 53,053 would otherwise allocate 22.5 GB)."""
    X = [np.asarray(s, dtype=np.float64) for s in series]
    N = len(X)
    stars = [None if (e is None or int(e) <= 0) else int(e) for e in e_star]
    groups: dict[int, list[int]] = {}
    for t, e in enumerate(stars):
        if e is not None:
            groups.setdefault(e, []).append(t)
    out = np.full((len(libraries), N), np.nan)
    for r, lib in enumerate(libraries):
        if stars[lib] is None:
            continue
        for E in sorted(groups):
            idx, w = knn_table(X[lib], E, tau, workers=workers)
            ids = groups[E]
            vals, _ = lookup(idx, w, E, tau, [X[t] for t in ids], workers=workers)
            for t, v in zip(ids, vals):
                if v is not None:
                    out[r, t] = v
    return out


def ccm_pairwise(series, E_max: int = 20, tau: int = 1, Tp: int = 1, workers=None):
    """ccm.py:94-151: per-series E* by edim, then xmap.  Returns (rho, e_star)."""
    stars = []
    for s in series:
        try:
            stars.append(edim(s, E_max, tau, Tp, workers)[0])
        except OracleError:
            raise
    rho, _ = xmap(series, stars, tau, workers)
    return rho, stars


# --------------------------------------------------------------------------
# library-size convergence sweep -- no reference implementation (parity unpinned)
# --------------------------------------------------------------------------

def sample_libraries(n_points: int, sizes, samples: int, seed: int):
    """Library samples for the convergence sweep.

    One ``np.random.default_rng(seed)`` PCG64 stream (the reference's RNG
    convention, synthetic.py:3-5); for each size in order, ``samples`` draws
    of ``rng.choice(n_points, size, replace=False)``, each sorted ascending.
    Sampling is WITHOUT replacement.  Returns a list (per size) of int64
    arrays [samples, size].
    """
    rng = np.random.default_rng(seed)
    out = []
    for L in sizes:
        L = int(L)
        if not 1 <= L <= n_points:
            raise OracleError("param", f"library size {L} outside [1, {n_points}]")
        out.append(np.stack([np.sort(rng.choice(n_points, L, replace=False))
                             for _ in range(samples)]).astype(np.int64))
    return out


def restricted_table(x, E: int, tau: int, lib_points: np.ndarray):
    """Neighbour table of every embedded point of x restricted to candidates in
    ``lib_points`` (self excluded, key (distance, point index), knn.py
    semantics), k = E + 1.  Returns (indices int64[n,k], weights f64[n,k])."""
    x = np.asarray(x, dtype=np.float64)
    n = point_count(x.size, E, tau)
    k = E + 1
    cand = np.asarray(lib_points, dtype=np.int64)
    D = np.zeros((n, cand.size))
    for e in range(E):
        a = x[e * tau: e * tau + n]
        diff = a[:, None] - a[cand][None, :]
        if e == 0:
            D = diff * diff
        else:
            D += diff * diff
    D[cand[None, :] == np.arange(n)[:, None]] = np.inf
    order = np.lexsort((np.broadcast_to(cand, D.shape), D), axis=1)[:, :k]
    idx = cand[order]
    d = np.take_along_axis(D, order, axis=1)
    if not np.all(np.isfinite(d)):
        raise OracleError("param", "library sample too small for k = E + 1 neighbours")
    return idx, simplex_weights(d)


def ccm_convergence(lib_series, tgt_series, E: int, tau: int, sizes, samples: int, seed: int):
    """Mean cross-map skill per library size (config 5 semantics, unpinned).

    For each size and sample: table restricted to the sampled library points,
    prediction of every embedded point of the target (Tp = 0), Pearson over
    all points; undefined skills are skipped in the mean (NaN if none).
    Returns float64[len(sizes)] of means and float64[len(sizes), samples]."""
    x = np.asarray(lib_series, dtype=np.float64)
    y = np.asarray(tgt_series, dtype=np.float64)
    n = valid_count(x.size, E, tau)
    libs = sample_libraries(n, sizes, samples, seed)
    per = np.full((len(sizes), samples), np.nan)
    for si, block in enumerate(libs):
        for s in range(samples):
            idx, w = restricted_table(x, E, tau, block[s])
            r, _ = lookup(idx, w, E, tau, [y], workers=1)
            if r[0] is not None:
                per[si, s] = r[0]
    with np.errstate(all="ignore"):
        means = np.array([np.nanmean(row) if np.any(np.isfinite(row)) else np.nan for row in per])
    return means, per


# ---------------------------------------------------------------- data formats
def skill_matrix_csv_bytes(names, rho) -> bytes:
    """write_skill_matrix (pkg/src/crossmap/io.py:66-78) restated: csv.writer rows
    ["", *names] then [name, *cells], cell = f"{v:.6f}" or "NA" when not finite,
    "\\r\\n" terminators.  Pinned by tests/golden/io_cases.json (reference output)."""
    import csv
    import io
    import math
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow([""] + list(names))
    for i, name in enumerate(names):
        w.writerow([name] + ["NA" if not math.isfinite(float(v)) else f"{float(v):.6f}" for v in rho[i]])
    return buf.getvalue().encode("utf-8")


class CsvOracleError(Exception):
    """The reference's CsvFormatError message (test oracle only)."""


def load_csv_rows(path):
    """load_csv (pkg/src/crossmap/io.py:25-61) restated on the csv module:
    (names, values[T][N]) or CsvOracleError(message)."""
    import csv
    import math
    with open(path, newline="", encoding="utf-8") as fh:
        rows = csv.reader(fh)
        try:
            head = next(rows)
        except StopIteration:
            raise CsvOracleError(f"{path}: empty file") from None
        names = [c.strip() for c in head]
        if not all(names):
            raise CsvOracleError(f"{path}: blank column name in header")
        dup = sorted({n for n in names if names.count(n) > 1})
        if dup:
            raise CsvOracleError(f"{path}: duplicate column names: {dup}")
        out = []
        for r, row in enumerate(rows, start=2):
            if len(row) != len(names):
                raise CsvOracleError(f"{path}: row {r} has {len(row)} cells, expected {len(names)}")
            vals = []
            for c, cell in enumerate(row):
                try:
                    v = float(cell)
                except ValueError:
                    raise CsvOracleError(f"{path}: row {r}, column {names[c]!r}: not numeric: {cell.strip()!r}") from None
                if not math.isfinite(v):
                    raise CsvOracleError(f"{path}: row {r}, column {names[c]!r}: non-finite value {cell.strip()!r}")
                vals.append(v)
            out.append(vals)
    if not names:
        raise IndexError("list index out of range")
    if not out:
        raise CsvOracleError(f"{path}: no data rows")
    return names, out


def read_skill_matrix_rows(path):
    """read_skill_matrix (io.py:81-110) restated: (names, rho) or CsvOracleError."""
    import csv
    with open(path, newline="", encoding="utf-8") as fh:
        rows = csv.reader(fh)
        try:
            head = next(rows)
        except StopIteration:
            raise CsvOracleError(f"{path}: empty file") from None
        names = head[1:]
        if not names:
            raise CsvOracleError(f"{path}: no target columns in header")
        rho = np.full((len(names), len(names)), np.nan)
        labels = []
        for r, row in enumerate(rows, start=2):
            if len(row) != len(names) + 1:
                raise CsvOracleError(f"{path}: row {r} has {len(row)} cells, expected {len(names) + 1}")
            labels.append(row[0])
            for c, cell in enumerate(row[1:]):
                if cell == "NA":
                    continue
                try:
                    rho[r - 2, c] = float(cell)
                except (ValueError, IndexError):
                    raise CsvOracleError(f"{path}: row {r}, column {names[c]!r}: bad cell {cell!r}") from None
    if labels != names:
        raise CsvOracleError(f"{path}: library rows do not match target columns")
    fin = rho[np.isfinite(rho)]
    if fin.size and (fin.min() < -1.0 or fin.max() > 1.0):  # SkillMatrix (ccm.py:65-74)
        raise OracleError("param", "finite skill entries must lie in [-1, 1]")
    return names, rho
