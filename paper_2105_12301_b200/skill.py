"""Simplex prediction and Pearson skill on the B200.

API mirror of pkg/src/crossmap/prediction.py:25-262.  ``lookup_batch`` and
``simplex_self_predict`` run gather + weighted sum + Pearson on the GPU;
``optimal_embedding`` runs the fused E = 1..E_max sweep (one kernel pass
over the candidates, every dimension's neighbour list maintained at once,
skill folded in-kernel) followed by the argmax.  ``PearsonAggregate`` keeps
the reference's mergeable-state interface; its ``from_arrays`` reduction runs
on the device, ``merge``/``correlation`` are O(1) scalar host logic.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import sqrt

import numpy as np

from . import _native as nat
from .embedding import DEFAULT_E_MAX, EmbeddingSpec, as_values, valid_count
from .errors import ParameterError, SeriesTooShortError, ZeroVarianceError
from .tables import NeighborTable

#: prediction.py:22 -- block size of the streamed aggregates
BLOCK = 4096


@dataclass(frozen=True)
class PearsonAggregate:
    """(count, means, second moments, co-moment); merges with the pooled rule."""

    count: int
    mean_a: float
    mean_b: float
    m2_a: float
    m2_b: float
    comoment: float

    @classmethod
    def empty(cls) -> "PearsonAggregate":
        return cls(0, 0.0, 0.0, 0.0, 0.0, 0.0)

    @classmethod
    def from_arrays(cls, a, b) -> "PearsonAggregate":
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel())
        b = np.ascontiguousarray(np.asarray(b, dtype=np.float64).ravel())
        if a.size != b.size:
            raise ParameterError(f"length mismatch: {a.size} vs {b.size}")
        if a.size == 0:
            return cls.empty()
        out = np.empty(6)
        nat.call("cmb_pearson", nat.device(), nat.ptr(a), nat.ptr(b), a.size, nat.ptr(out))
        return cls(int(out[0]), float(out[1]), float(out[2]), float(out[3]), float(out[4]), float(out[5]))

    def merge(self, other: "PearsonAggregate") -> "PearsonAggregate":
        if self.count == 0:
            return other
        if other.count == 0:
            return self
        n = self.count + other.count
        da = other.mean_a - self.mean_a
        db = other.mean_b - self.mean_b
        f = self.count * other.count / n
        return PearsonAggregate(n, self.mean_a + da * other.count / n, self.mean_b + db * other.count / n,
                                self.m2_a + other.m2_a + da * da * f, self.m2_b + other.m2_b + db * db * f,
                                self.comoment + other.comoment + da * db * f)

    def correlation(self) -> float | None:
        if self.count < 2 or self.m2_a <= 0.0 or self.m2_b <= 0.0:
            return None
        return float(min(1.0, max(-1.0, self.comoment / sqrt(self.m2_a * self.m2_b))))


def pearson_stream(a, b) -> float:
    """Pearson correlation via 4096-point device aggregates; ZeroVarianceError if undefined."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 1 or b.ndim != 1:
        raise ParameterError("correlation inputs must be 1-D")
    if a.size != b.size:
        raise ParameterError(f"length mismatch: {a.size} vs {b.size}")
    if a.size < 2:
        raise ParameterError("correlation needs at least 2 observations")
    rho = PearsonAggregate.from_arrays(a, b).correlation()
    if rho is None:
        raise ZeroVarianceError("correlation undefined: an input has zero variance")
    return rho


@dataclass(frozen=True, eq=False)
class PredictionOutput:
    """Skill (None when undefined) and, on request, the predicted series."""

    rho: float | None
    predicted: np.ndarray | None = None

    @property
    def defined(self) -> bool:
        return self.rho is not None


def lookup_batch(table: NeighborTable, targets, want_predictions: bool = False,
                 workers: int | None = None) -> list[PredictionOutput]:
    """Cross-map every target through one neighbour table (float64 device kernel)."""
    ys = [np.ascontiguousarray(as_values(t)) for t in targets]
    off = table.spec.span
    n = table.n
    for t, y in enumerate(ys):
        if y.size < n + off:
            raise ParameterError(f"target {t} has {y.size} samples; table needs at least {n + off}")
    out: list[PredictionOutput | None] = [None] * len(ys)
    if not ys:
        return []
    idx = np.ascontiguousarray(table.indices, dtype=np.int64)
    w = np.ascontiguousarray(table.weights, dtype=np.float64)
    by_len: dict[int, list[int]] = {}
    for t, y in enumerate(ys):
        by_len.setdefault(y.size, []).append(t)
    for length, ids in by_len.items():
        Y = np.ascontiguousarray(np.stack([ys[t] for t in ids]))
        rho = np.empty(len(ids))
        pred = np.empty((len(ids), n)) if want_predictions else None
        nat.call("cmb_lookup", nat.device(), nat.ptr(idx), nat.ptr(w), n, table.k, off,
                 nat.ptr(Y), length, len(ids), nat.ptr(rho), nat.ptr(pred))
        for q, t in enumerate(ids):
            r = None if np.isnan(rho[q]) else float(rho[q])
            out[t] = PredictionOutput(r, pred[q].copy() if pred is not None else None)
    return out  # type: ignore[return-value]


# Widest dimension of the fused sweep kernels (CMB_SWEEP_MAX_E in csrc/cmb_common.cuh).
# Larger E (the reference accepts any e_max) runs the reference's own composition
# -- build_knn_table + lookup_batch, both device kernels -- one (series, E) at a time.
NATIVE_E_MAX = 30


def _simplex_composed(v: np.ndarray, spec: EmbeddingSpec, tp: int) -> float:
    """prediction.py:178-179: table on v[:len - tp], lookup of v[tp:]; NaN = undefined."""
    from .tables import build_knn_table
    table = build_knn_table(v[: v.size - tp], spec)
    r = lookup_batch(table, [v[tp:]])[0].rho
    return float("nan") if r is None else r


def simplex_self_predict(series, spec: EmbeddingSpec, tp: int = 1, workers: int | None = None) -> float:
    """Skill of forecasting a series tp steps ahead from its own manifold."""
    v = np.ascontiguousarray(as_values(series))
    if tp < 1:
        raise ParameterError(f"prediction horizon must be >= 1, got {tp}")
    if v.size <= tp:
        raise SeriesTooShortError(f"series of length {v.size} cannot support horizon {tp}")
    valid_count(v.size - tp, spec)
    rho = np.empty(1)
    if spec.E > NATIVE_E_MAX:
        rho[0] = _simplex_composed(v, spec, tp)
    else:
        nat.call("cmb_simplex", nat.device(), nat.ptr(v), v.size, spec.E, spec.tau, tp, nat.ptr(rho))
    if np.isnan(rho[0]):
        raise ZeroVarianceError("self-prediction skill undefined: constant values over the forecast range")
    return float(rho[0])


@dataclass(frozen=True)
class OptimalEmbedding:
    """Best dimension and the whole skill curve {E: rho}."""

    e_star: int
    rho_by_e: dict

    def __post_init__(self):
        if self.e_star not in self.rho_by_e:
            raise ParameterError(f"optimal dimension {self.e_star} missing from the skill curve")


def skill_curves(X: np.ndarray, e_max: int, tau: int, tp: int) -> tuple[np.ndarray, np.ndarray]:
    """Batched device edim: X (series, time) -> (rho[N, e_max] NaN = undefined,
    e_star[N] with 0 = undefined)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    N, L = X.shape
    rho = np.empty((N, e_max))
    est = np.empty(N, dtype=np.int32)
    if e_max > NATIVE_E_MAX:
        _edim_wide(X, e_max, tau, tp, rho, est)
    else:
        nat.call("cmb_edim", nat.device(), nat.ptr(X), N, L, e_max, tau, tp, nat.ptr(rho), nat.ptr(est))
    return rho, est


def near_ties(rho: np.ndarray, est: np.ndarray, tol: float = 1e-4) -> list[dict]:
    """Series whose E* is fragile: the best curve value and the runner-up differ
    by less than ``tol`` (SURVEY.md 8c parity rule: E* identical to the
    reference's except logged curve near-ties; prediction.py:258-261 takes the
    first maximum).  One dict per such series: series, e_star, runner_up, gap."""
    out = []
    rho = np.asarray(rho, dtype=np.float64)
    for s in np.flatnonzero(np.asarray(est) > 0):
        curve = rho[s]
        b = int(est[s]) - 1
        others = np.delete(curve, b)
        idx = np.delete(np.arange(curve.size), b)
        r = int(np.argmax(others))
        gap = float(curve[b] - others[r])
        if gap < tol:
            out.append({"series": int(s), "e_star": b + 1, "runner_up": int(idx[r]) + 1, "gap": gap})
    return out


def _edim_wide(X: np.ndarray, e_max: int, tau: int, tp: int, rho: np.ndarray, est: np.ndarray) -> None:
    """skill_curves for e_max > NATIVE_E_MAX: the fused sweep for E <= NATIVE_E_MAX, the
    reference composition per (series, E) above it, E* re-taken over the whole curve
    (strict >, ties to the smaller E; undefined when any E is undefined, ccm.py:113-121)."""
    N, L = X.shape
    part = np.empty((N, NATIVE_E_MAX))
    est_dev = np.empty(N, dtype=np.int32)
    nat.call("cmb_edim", nat.device(), nat.ptr(X), N, L, NATIVE_E_MAX, tau, tp, nat.ptr(part), nat.ptr(est_dev))
    rho[:, :NATIVE_E_MAX] = part
    for s in range(N):
        v = X[s]
        for E in range(NATIVE_E_MAX + 1, e_max + 1):
            rho[s, E - 1] = (_simplex_composed(v, EmbeddingSpec(E, tau, e_max=e_max), tp)
                             if v.min() != v.max() else np.nan)
        curve = rho[s]
        if est_dev[s] == 0 or np.isnan(curve).any():
            est[s] = 0
            continue
        best = 0
        for e in range(1, e_max):
            if curve[e] > curve[best]:
                best = e
        est[s] = best + 1


def optimal_embedding(series, e_max: int = DEFAULT_E_MAX, tau: int = 1, tp: int = 1,
                      workers: int | None = None) -> OptimalEmbedding:
    """Self-prediction skill for E in [1, e_max]; the best E wins, ties to the smaller E."""
    v = as_values(series)
    if e_max < 1:
        raise ParameterError(f"dimension bound must be >= 1, got {e_max}")
    if tp < 1:
        raise ParameterError(f"prediction horizon must be >= 1, got {tp}")
    if v.min() == v.max():
        raise ZeroVarianceError("cannot search embeddings of a constant series")
    if v.size <= tp:
        raise SeriesTooShortError(f"series of length {v.size} cannot support horizon {tp}")
    valid_count(v.size - tp, EmbeddingSpec(e_max, tau, e_max=e_max))
    rho, est = skill_curves(v[None, :], e_max, tau, tp)
    bad = np.flatnonzero(np.isnan(rho[0]))
    if bad.size:
        raise ZeroVarianceError(
            f"self-prediction skill undefined at E={int(bad[0]) + 1}: constant values over the forecast range")
    return OptimalEmbedding(int(est[0]), {e + 1: float(rho[0, e]) for e in range(e_max)})
