"""Library-size convergence sweep (kEDM ``ccm``) on the B200.

The reference package stops at the all-to-all cross map ("no
convergence sweep over library sizes ... in v1"); this is the next row of the
hot-path scope.  Semantics (also restated in the
oracle, oracle/crossmap_oracle.py ``ccm_convergence``; parity with the
reference is necessarily UNPINNED):

* library samples: one ``np.random.default_rng(seed)`` PCG64 stream (the
  reference's RNG convention, synthetic.py:3-5); for each library size in
  order, ``samples`` draws of ``rng.choice(n_E, size, replace=False)``, each
  sorted -- sampling WITHOUT replacement over embedded points;
* neighbours: every embedded point of the library is matched to its E + 1
  nearest points of the sample (self excluded, ties to the lower index,
  knn.py semantics), simplex weights per knn.py:180-202;
* skill: every embedded point of the target is predicted (Tp = 0) and scored
  with Pearson; undefined skills are NaN and skipped by the means.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as nat
from .embedding import as_values, valid_count, EmbeddingSpec
from .errors import ParameterError


def sample_libraries(n_points: int, sizes: Sequence[int], samples: int, seed: int) -> list:
    """Seeded library samples: per size an int32 array [samples, size] of sorted point indices."""
    rng = np.random.default_rng(seed)
    out = []
    for L in sizes:
        L = int(L)
        if not 1 <= L <= n_points:
            raise ParameterError(f"library size {L} outside [1, {n_points}]")
        out.append(np.stack([np.sort(rng.choice(n_points, L, replace=False)) for _ in range(samples)])
                   .astype(np.int32))
    return out


@dataclass(frozen=True)
class Convergence:
    """Skill per library size: ``mean`` [sizes], ``rho`` [sizes, samples] (NaN undefined)."""

    sizes: np.ndarray
    mean: np.ndarray
    rho: np.ndarray


def _means(rho: np.ndarray) -> np.ndarray:
    ok = np.isfinite(rho)
    cnt = ok.sum(axis=-1)
    tot = np.where(ok, rho, 0.0).sum(axis=-1)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(cnt > 0, tot / np.maximum(cnt, 1), np.nan)


def ccm_sweep(values, E, lib_sizes: Sequence[int], samples: int = 100, tau: int = 1, seed: int = 0,
              pairs: Sequence[tuple[int, int]] | None = None) -> np.ndarray:
    """Convergence sweep over (library, target) pairs of the columns of ``values`` (time, series).

    ``E``: scalar or per-target embedding dimensions (the library is embedded at
    the target's E, as in xmap).  ``pairs`` defaults to every ordered pair.
    Returns rho float64 [P, len(lib_sizes), samples] in pair order.
    """
    X = np.ascontiguousarray(np.asarray(values, dtype=np.float64).T)
    N, T = X.shape
    if not np.all(np.isfinite(X)):
        raise ParameterError("non-finite observation in the sweep input")
    Es = np.full(N, int(E), dtype=np.int32) if np.ndim(E) == 0 else np.asarray(E, dtype=np.int32)
    if Es.size != N:
        raise ParameterError(f"{Es.size} dimensions for {N} series")
    if pairs is None:
        pairs = [(l, t) for l in range(N) for t in range(N)]
    pairs = [(int(l), int(t)) for l, t in pairs]
    sizes = np.asarray(lib_sizes, dtype=np.int32)
    if samples < 1:
        raise ParameterError("samples must be >= 1")
    out = np.full((len(pairs), sizes.size, samples), np.nan)
    by_e: dict[int, list[int]] = {}
    for p, (_, t) in enumerate(pairs):
        by_e.setdefault(int(Es[t]), []).append(p)
    for e, plist in sorted(by_e.items()):
        n = valid_count(T, EmbeddingSpec(e, tau, e_max=max(e, 20)))
        pts = sample_libraries(n, sizes, samples, seed)
        flat = np.ascontiguousarray(np.concatenate([b.ravel() for b in pts]).astype(np.int32))
        lib = np.ascontiguousarray([pairs[p][0] for p in plist], dtype=np.int32)
        tgt = np.ascontiguousarray([pairs[p][1] for p in plist], dtype=np.int32)
        rho = np.empty((len(plist), sizes.size, samples))
        nat.call("cmb_ccm_convergence", nat.device(), nat.ptr(X), N, T, e, tau, nat.ptr(lib),
                 nat.ptr(tgt), len(plist), nat.ptr(np.ascontiguousarray(sizes)), sizes.size, samples,
                 nat.ptr(flat), nat.ptr(rho))
        out[plist] = rho
    return out


def ccm(library, target, E: int, lib_sizes: Sequence[int], samples: int = 100, tau: int = 1,
        seed: int = 0) -> Convergence:
    """Convergent cross mapping skill of ``target`` from ``library``'s manifold vs library size."""
    x = as_values(library)
    y = as_values(target)
    if x.size != y.size:
        raise ParameterError(f"series lengths differ: {x.size} vs {y.size}")
    rho = ccm_sweep(np.stack([x, y], axis=1), [E, E], lib_sizes, samples, tau, seed, pairs=[(0, 1)])[0]
    return Convergence(np.asarray(lib_sizes, dtype=np.int64), _means(rho), rho)
