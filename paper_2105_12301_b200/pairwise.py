"""All-to-all cross mapping (xmap) on the B200.

API mirror of pkg/src/crossmap/ccm.py:25-151.  ``ccm_pairwise`` runs the
batched edim sweep for every series at once (one kernel launch per batch of
series instead of N serial calls), groups targets by E*, and hands the whole
N x N problem to ``cmb_xmap``: per library one sweep emits every needed
dimension's table, and the lookup kernel crosses each table with every target
of the matching group, writing only rho.

Precision: neighbour selection is exact (fp64-certified); tables store fp32
weights and the lookup accumulates in fp32 with fp64 folds, so rho agrees with
the float64 reference to ~1e-6 (north-star tolerance 1e-4).
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as nat
from .embedding import DEFAULT_E_MAX, Dataset, EmbeddingSpec
from .errors import ParameterError
from .skill import NATIVE_E_MAX, OptimalEmbedding, lookup_batch, skill_curves
from .tables import build_knn_table

LAYOUT_LIB_MAJOR = 0
LAYOUT_TGT_MAJOR = 1


@dataclass(frozen=True)
class CcmConfig:
    """Pipeline parameters (ccm.py:25-40)."""

    e_max: int = DEFAULT_E_MAX
    tau: int = 1
    tp_search: int = 1
    emit_predictions: bool = False

    def __post_init__(self):
        for name, val in (("e_max", self.e_max), ("tau", self.tau), ("tp_search", self.tp_search)):
            if val < 1:
                raise ParameterError(f"{name} must be >= 1, got {val}")


@dataclass
class CcmStats:
    """Phase timings and scheduling counters of one run (ccm.py:43-53)."""

    seconds_optimal_e: float = 0.0
    seconds_table_build: float = 0.0
    seconds_lookup: float = 0.0
    tables_built: int = 0
    distinct_e: int = 0
    n_series: int = 0
    series_length: int = 0


@dataclass(frozen=True, eq=False)
class SkillMatrix:
    """rho[library, target]; NaN marks undefined skill (ccm.py:56-83)."""

    names: list
    rho: np.ndarray
    stats: CcmStats | None = None
    predictions: dict | None = None

    def __post_init__(self):
        m = np.asarray(self.rho, dtype=np.float64)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ParameterError(f"skill matrix must be square, got shape {m.shape}")
        if len(self.names) != m.shape[0]:
            raise ParameterError(f"{len(self.names)} names for a {m.shape[0]}-row matrix")
        fin = m[np.isfinite(m)]
        if fin.size and (fin.min() < -1.0 or fin.max() > 1.0):
            raise ParameterError("finite skill entries must lie in [-1, 1]")
        object.__setattr__(self, "rho", m)
        object.__setattr__(self, "names", list(self.names))

    @property
    def n(self) -> int:
        return self.rho.shape[0]

    @property
    def defined(self) -> np.ndarray:
        return np.isfinite(self.rho)


def group_by_optimal_e(embeddings: Sequence[OptimalEmbedding]) -> dict:
    """Series positions keyed by their optimal dimension (ccm.py:86-91)."""
    groups: dict = {}
    for pos, emb in enumerate(embeddings):
        groups.setdefault(emb.e_star, []).append(pos)
    return groups


def xmap(values, e_star, tau: int = 1, layout: int = LAYOUT_LIB_MAJOR, dtype=np.float64,
         stats: dict | None = None) -> np.ndarray:
    """rho over all ordered pairs of the columns of ``values`` (time, series).

    ``e_star[j]`` is the embedding dimension of target j (0 or None = undefined
    series: NaN row and column).  Returns rho[lib, tgt]; with
    ``layout=LAYOUT_TGT_MAJOR`` the same matrix is returned as an
    F-ordered view of the kernel's native target-major buffer (no transpose
    pass).  ``dtype`` float32 skips the float64 widening.
    """
    X = np.asarray(values)
    if X.ndim != 2:
        raise ParameterError(f"expected a 2-D (time, series) array, got shape {X.shape}")
    T, N = X.shape
    est = np.array([0 if (e is None or int(e) <= 0) else int(e) for e in e_star], dtype=np.int32)
    if est.size != N:
        raise ParameterError(f"{est.size} dimensions for {N} series")
    if tau < 1:
        raise ParameterError(f"tau must be >= 1, got {tau}")
    # float32 input runs the float32 entry; anything else is staged in float64
    # (the reference's dtype, series.py:25): cmb_xmap64 centres each series in
    # fp64 before the fp32 sweep and certifies neighbours against the fp64 values
    f32 = X.dtype == np.float32
    Xs = np.ascontiguousarray(X.T, dtype=np.float32 if f32 else np.float64)  # series-major samples
    # beyond the fused kernels' formats (E* > NATIVE_E_MAX, or T past the 16-bit
    # row indices of the table records) the affected pairs take the reference's
    # composition on the device: build_knn_table + lookup_batch per (library, E)
    wide = (est > NATIVE_E_MAX) | ((T > NATIVE_T_MAX) & (est > 0))
    if wide.any():
        return _xmap_with_wide(np.ascontiguousarray(Xs, dtype=np.float32), est, wide, tau, layout, dtype, stats)
    out = nat.host_empty((N, N), np.float32)
    st = np.zeros(8)
    nat.call("cmb_xmap" if f32 else "cmb_xmap64", nat.device(), nat.ptr(Xs), N, T, nat.ptr(est), tau,
             nat.ptr(out), layout, nat.ptr(st))
    if stats is not None:
        stats.update(seconds_table_build=float(st[0]), seconds_lookup=float(st[1]),
                     seconds_total=float(st[2]), tables_built=int(st[3]), distinct_e=int(st[4]),
                     pairs=int(st[5]))
    rho = out.T if layout == LAYOUT_TGT_MAJOR else out
    return rho.astype(dtype, copy=False) if dtype != np.float32 else rho


NATIVE_T_MAX = 65535  # 16-bit neighbour rows in the cross-map table records (csrc/cmb_common.cuh)


def xmap_predictions(values, e_star, pairs, tau: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """The cross map plus materialised predictions of the (library, target)
    ``pairs`` (lookup_batch(want_predictions=True), prediction.py:145-153) from
    the same device tables and targets as rho (cmb_xmap_predict).  Returns
    (rho[lib, tgt] float32, pred float32 [len(pairs), T]; row p holds target
    pairs[p][1]'s prediction at its n_E embedded points, NaN after them and for
    pairs with an undefined series)."""
    X = np.asarray(values, dtype=np.float64)
    T, N = X.shape
    est = np.array([0 if (e is None or int(e) <= 0) else int(e) for e in e_star], dtype=np.int32)
    if est.size != N:
        raise ParameterError(f"{est.size} dimensions for {N} series")
    pl = np.ascontiguousarray([p[0] for p in pairs], dtype=np.int32)
    pt = np.ascontiguousarray([p[1] for p in pairs], dtype=np.int32)
    Xs = np.ascontiguousarray(X.T)
    rho = nat.host_empty((N, N), np.float32)
    pred = nat.host_empty((max(pl.size, 1), T), np.float32)
    nat.call("cmb_xmap_predict", nat.device(), nat.ptr(Xs), N, T, nat.ptr(est), tau, nat.ptr(pl), nat.ptr(pt),
             pl.size, nat.ptr(rho), LAYOUT_LIB_MAJOR, nat.ptr(pred), None)
    return rho, pred[: pl.size]


def _xmap_with_wide(Xs: np.ndarray, est: np.ndarray, wide: np.ndarray, tau: int, layout: int, dtype,
                    stats: dict | None) -> np.ndarray:
    """xmap when some targets are outside the fused kernels' formats.  The fused
    path runs with those series masked (which also drops them as libraries); the
    masked libraries' rows for the other targets and every library's column for
    a wide target are then computed per (library, E) with build_knn_table +
    lookup_batch (float64 device kernels, ccm.py:131-149 semantics)."""
    N, T = Xs.shape
    t0 = time.perf_counter()
    rho = np.full((N, N), np.nan)
    est_n = np.where(wide, 0, est).astype(np.int32)
    st = np.zeros(8)
    if (est_n > 0).any():
        out = np.empty((N, N), dtype=np.float32)
        nat.call("cmb_xmap", nat.device(), nat.ptr(Xs), N, T, nat.ptr(est_n), tau, nat.ptr(out),
                 LAYOUT_LIB_MAJOR, nat.ptr(st))
        rho[:] = out
    narrow: dict = {}
    far: dict = {}
    for t in np.flatnonzero(est > 0):
        (far if wide[t] else narrow).setdefault(int(est[t]), []).append(int(t))
    X64 = Xs.astype(np.float64)
    e_top = max(int(est.max()), 1)
    for lib in np.flatnonzero(est > 0):
        groups = dict(far)
        if wide[lib]:
            for e, ts in narrow.items():
                groups[e] = groups.get(e, []) + ts
        for e in sorted(groups):
            ts = groups[e]
            table = build_knn_table(X64[lib], EmbeddingSpec(e, tau, e_max=e_top))
            outs = lookup_batch(table, [X64[t] for t in ts])
            rho[lib, ts] = [np.nan if o.rho is None else o.rho for o in outs]
    if stats is not None:
        stats.update(seconds_table_build=float(st[0]), seconds_lookup=float(st[1]),
                     seconds_total=time.perf_counter() - t0, tables_built=int(st[3]), distinct_e=int(st[4]),
                     pairs=int(np.sum(est > 0)) ** 2)
    out = rho.astype(dtype, copy=False)
    return np.asfortranarray(out) if layout == LAYOUT_TGT_MAJOR else out


def ccm_pairwise(data: Dataset, cfg: CcmConfig | None = None, workers: int | None = None,
                 e_star: Sequence[int] | None = None) -> SkillMatrix:
    """Full N x N cross-map skill matrix, diagonal included (ccm.py:94-151)."""
    cfg = cfg or CcmConfig()
    n = len(data)
    stats = CcmStats(n_series=n, series_length=data.length)
    X = data.matrix()
    if e_star is not None:
        if len(e_star) != n:
            raise ParameterError(f"{len(e_star)} dimension overrides for {n} series")
        stars = []
        for e in e_star:
            if not 1 <= int(e) <= cfg.e_max:
                raise ParameterError(f"dimension override {e} outside [1, {cfg.e_max}]")
            stars.append(int(e))
    else:
        t0 = time.perf_counter()
        # the reference's per-series guards (prediction.py:249-256) apply to the batch
        EmbeddingSpec(cfg.e_max, cfg.tau, e_max=cfg.e_max)
        _, est = skill_curves(X, cfg.e_max, cfg.tau, cfg.tp_search)
        stars = [int(e) if e > 0 else None for e in est]
        stats.seconds_optimal_e = time.perf_counter() - t0
    groups: dict = {}
    for i, s in enumerate(stars):
        if s is not None:
            groups.setdefault(s, []).append(i)
    stats.distinct_e = len(groups)
    info: dict = {}
    est = [s or 0 for s in stars]
    predictions = None
    native = max(est) <= NATIVE_E_MAX and data.length <= NATIVE_T_MAX
    if cfg.emit_predictions and native:
        # every defined (library, target) pair, in the reference's order
        # (ccm.py:131-149: library, then E group, then target)
        order = [(lib, t) for lib in range(n) if stars[lib] is not None
                 for e in sorted(groups) for t in groups[e]]
        t0 = time.perf_counter()
        rho32, pred = xmap_predictions(X.T, est, order, cfg.tau)
        rho = rho32.astype(np.float64)
        info["seconds_lookup"] = time.perf_counter() - t0
        predictions = {}
        for p, (lib, t) in enumerate(order):
            ne = data.length - (stars[t] - 1) * cfg.tau
            predictions[(lib, t)] = pred[p, :ne].astype(np.float64)
    else:
        rho = xmap(X.T, est, cfg.tau, layout=LAYOUT_TGT_MAJOR, stats=info)
        if cfg.emit_predictions:  # formats past the fused kernels: the device composition per (library, E)
            predictions = {}
            for lib in range(n):
                if stars[lib] is None:
                    continue
                for e in sorted(groups):
                    table = build_knn_table(data[lib], EmbeddingSpec(e, cfg.tau, e_max=cfg.e_max))
                    outs = lookup_batch(table, [data[t] for t in groups[e]], want_predictions=True)
                    for t, o in zip(groups[e], outs):
                        if o.predicted is not None:
                            predictions[(lib, t)] = o.predicted
    stats.seconds_table_build = info.get("seconds_table_build", 0.0)
    stats.seconds_lookup = info.get("seconds_lookup", 0.0)
    stats.tables_built = sum(1 for s in stars if s is not None) * len(groups)
    return SkillMatrix(data.names, rho, stats=stats, predictions=predictions)
