"""Neighbour tables over delay embeddings, computed on the B200.

API mirror of pkg/src/crossmap/knn.py:30-252.  ``build_knn_table`` runs the
fused sweep kernel (csrc/knn_sweep.cu): the n x n distance matrix is never
materialised, selection is exact (fp64-certified, ties to the lower index)
and weights follow knn.py:180-202.  The reference's materialised primitives
(``pairwise_distances``, ``partial_sort_topk``, ``normalize_to_weights``)
are provided on the GPU as well, with the same semantics, for callers that
use them directly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .embedding import EmbeddingSpec, as_values, valid_count
from .errors import ParameterError, SeriesTooShortError

#: knn.py:27 -- floor of exp() weights
TINY = np.finfo(np.float64).tiny


@dataclass(frozen=True, eq=False)
class DistanceMatrix:
    """Square matrix of squared Euclidean distances between embedded points."""

    values: np.ndarray

    def __post_init__(self):
        m = np.asarray(self.values, dtype=np.float64)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ParameterError(f"distance matrix must be square, got shape {m.shape}")
        if np.any(np.diagonal(m) != 0.0):
            raise ParameterError("distance matrix diagonal must be exactly zero")
        object.__setattr__(self, "values", m)

    @property
    def n(self) -> int:
        return self.values.shape[0]


@dataclass(frozen=True, eq=False)
class NeighborTable:
    """Row i: the k nearest embedded points to point i (self excluded), ascending,
    with simplex weights summing to 1.  Validation rules of knn.py:63-86."""

    indices: np.ndarray
    weights: np.ndarray
    spec: EmbeddingSpec

    def __post_init__(self):
        idx = np.asarray(self.indices)
        w = np.asarray(self.weights, dtype=np.float64)
        if idx.ndim != 2 or idx.shape != w.shape:
            raise ParameterError(f"indices {idx.shape} and weights {w.shape} must be matching 2-D arrays")
        n, k = idx.shape
        if not np.issubdtype(idx.dtype, np.integer):
            raise ParameterError("neighbor indices must be integers")
        if idx.size and (idx.min() < 0 or idx.max() >= n):
            raise ParameterError(f"neighbor indices must lie in [0, {n})")
        if (idx == np.arange(n)[:, None]).any():
            raise ParameterError("a point may not be its own neighbor")
        if k > 1 and (np.diff(np.sort(idx, axis=1), axis=1) == 0).any():
            raise ParameterError("neighbor indices must be distinct per row")
        if ((w <= 0.0) | (w > 1.0)).any():
            raise ParameterError("weights must lie in (0, 1]")
        if (np.abs(w.sum(axis=1) - 1.0) > 1e-6).any():
            raise ParameterError("weight rows must sum to 1")
        if k > 1 and (np.diff(w, axis=1) > 1e-12).any():
            raise ParameterError("weight rows must be non-increasing")
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "weights", w)

    @property
    def n(self) -> int:
        return self.indices.shape[0]

    @property
    def k(self) -> int:
        return self.indices.shape[1]


def pairwise_distances(series, spec: EmbeddingSpec, workers: int | None = None) -> DistanceMatrix:
    """All squared delay-vector distances of one series (GPU, reference op order)."""
    v = np.ascontiguousarray(as_values(series))
    n = spec.point_count(v.size)
    if n < 2:
        raise SeriesTooShortError(
            f"series of length {v.size} yields {n} embedded points for E={spec.E}, "
            f"tau={spec.tau}; pairwise distances need at least 2")
    out = np.empty((n, n))
    nat.call("cmb_pairwise_distances", nat.device(), nat.ptr(v), v.size, spec.E, spec.tau, nat.ptr(out))
    return DistanceMatrix(out)


def partial_sort_topk(distances, k: int, workers: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Per row the k smallest entries over j != i, ordered by (value, column)."""
    m = distances.values if isinstance(distances, DistanceMatrix) else np.asarray(distances, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ParameterError(f"expected a square distance matrix, got shape {m.shape}")
    n = m.shape[0]
    if not 1 <= k <= n - 1:
        raise ParameterError(f"neighbor count must lie in [1, {n - 1}], got {k}")
    m = np.ascontiguousarray(m)
    d = np.empty((n, k))
    i = np.empty((n, k), dtype=np.int64)
    nat.call("cmb_partial_sort_topk", nat.device(), nat.ptr(m), n, k, nat.ptr(d), nat.ptr(i))
    return d, i


def normalize_to_weights(top_squared) -> np.ndarray:
    """Simplex weights exp(-d/dmin), normalised, from ascending squared distances."""
    sq = np.ascontiguousarray(np.asarray(top_squared, dtype=np.float64))
    if sq.ndim != 2:
        raise ParameterError(f"expected an n x k distance array, got shape {sq.shape}")
    out = np.empty_like(sq)
    if sq.size:
        nat.call("cmb_normalize_weights", nat.device(), nat.ptr(sq), sq.shape[0], sq.shape[1], nat.ptr(out))
    return out


def _table_arrays(v: np.ndarray, spec: EmbeddingSpec, k: int):
    n = spec.point_count(v.size)
    if not 1 <= k <= n - 1:
        raise ParameterError(f"neighbor count must lie in [1, {n - 1}], got {k}")
    idx = np.empty((n, k), dtype=np.int64)
    w = np.empty((n, k))
    d = np.empty((n, k))
    nat.call("cmb_knn_table", nat.device(), nat.ptr(v), v.size, spec.E, spec.tau, k,
             nat.ptr(idx), nat.ptr(w), nat.ptr(d))
    return idx, w, d


def build_knn_table(series, spec: EmbeddingSpec, k: int | None = None,
                    workers: int | None = None) -> NeighborTable:
    """Fused embedding + distance + exact top-k + weights (k defaults to E + 1)."""
    v = np.ascontiguousarray(as_values(series))
    valid_count(v.size, spec)
    idx, w, _ = _table_arrays(v, spec, spec.E + 1 if k is None else k)
    return NeighborTable(idx, w, spec)


def oracle_knn(series, spec: EmbeddingSpec, k: int | None = None) -> NeighborTable:
    """The reference's transparent builder (knn.py:220-252), here the materialised
    GPU path: full distance matrix, full per-row sort, direct weights."""
    v = np.ascontiguousarray(as_values(series))
    n = valid_count(v.size, spec)
    k = spec.E + 1 if k is None else k
    if not 1 <= k <= n - 1:
        raise ParameterError(f"neighbor count must lie in [1, {n - 1}], got {k}")
    d, i = partial_sort_topk(pairwise_distances(v, spec), k)
    return NeighborTable(i, normalize_to_weights(d), spec)
