"""Kernel micro-benchmarks: (E, phase, seconds) rows over a dimension sweep.

Drop-in for the reference harness (pkg/src/crossmap/bench.py:1-91: same
``run_bench`` signature, row shape, desk-scale bounds and CSV text), timing
this package's device-backed API on seeded synthetic data, so the paper's
Figures 2-5-style sweeps can be regenerated on a B200:

* ``knn``: per E, "distance" = ``pairwise_distances`` (the materialised fp64
  distance kernel) and "topk" = ``partial_sort_topk`` (CTA bitonic selection)
  -- the reference's two phases; ``fused=True`` adds a "fused" row, the
  production path (``build_knn_table``: distances, exact top-(E+1) and weights
  in one sweep that never materialises the matrix).
* ``lookup``: per E, one table on a library series, then ``lookup_batch`` over
  ``count`` targets.

Each call is synchronous, so wall-clock phase times include the host<->device
copies of the public API (the reference's times include its whole functions).
"""

from __future__ import annotations

import io
from dataclasses import dataclass
from time import perf_counter

import numpy as np

from .embedding import DEFAULT_E_MAX, EmbeddingSpec
from .errors import ParameterError
from .skill import lookup_batch
from .tables import build_knn_table, pairwise_distances, partial_sort_topk

DESK_MAX_LENGTH = 10_000
DESK_MAX_SERIES = 10_000

KINDS = ("knn", "lookup")


@dataclass(frozen=True)
class BenchRow:
    e: int
    phase: str
    seconds: float


def run_bench(kind: str, length: int = 4000, count: int = 1000,
              e_range: tuple[int, int] = (1, DEFAULT_E_MAX), seed: int = 0,
              workers: int | None = None, allow_large: bool = False,
              fused: bool = False) -> list[BenchRow]:
    """Time one kernel family across an embedding-dimension sweep (bench.py:34-83).

    ``workers`` is accepted for signature compatibility (the GPU grid replaces
    the reference's thread pool)."""
    if kind not in KINDS:
        raise ParameterError(f"unknown bench kind {kind!r}; choose from {KINDS}")
    e_lo, e_hi = int(e_range[0]), int(e_range[1])
    if not 1 <= e_lo <= e_hi:
        raise ParameterError(f"bad dimension range {e_range}")
    if not allow_large:
        if length > DESK_MAX_LENGTH:
            raise ParameterError(
                f"length {length} exceeds the desk-scale bound {DESK_MAX_LENGTH}; "
                f"pass allow_large to override")
        if kind == "lookup" and count > DESK_MAX_SERIES:
            raise ParameterError(
                f"target count {count} exceeds the desk-scale bound {DESK_MAX_SERIES}; "
                f"pass allow_large to override")
    bound = max(e_hi, DEFAULT_E_MAX)
    rng = np.random.default_rng(seed)
    rows: list[BenchRow] = []
    if kind == "knn":
        library = rng.random(length)
        for e in range(e_lo, e_hi + 1):
            spec = EmbeddingSpec(e, 1, e_max=bound)
            began = perf_counter()
            dmat = pairwise_distances(library, spec, workers=workers)
            mid = perf_counter()
            partial_sort_topk(dmat, e + 1, workers=workers)
            done = perf_counter()
            rows.append(BenchRow(e, "distance", mid - began))
            rows.append(BenchRow(e, "topk", done - mid))
            if fused:
                began = perf_counter()
                build_knn_table(library, spec, workers=workers)
                rows.append(BenchRow(e, "fused", perf_counter() - began))
    else:
        library = rng.random(length)
        targets = rng.random((count, length))
        for e in range(e_lo, e_hi + 1):
            spec = EmbeddingSpec(e, 1, e_max=bound)
            table = build_knn_table(library, spec, workers=workers)
            began = perf_counter()
            lookup_batch(table, list(targets), workers=workers)
            rows.append(BenchRow(e, "lookup", perf_counter() - began))
    return rows


def bench_rows_to_csv(rows: list[BenchRow]) -> str:
    out = io.StringIO()
    out.write("E,phase,seconds\n")
    for row in rows:
        out.write(f"{row.e},{row.phase},{row.seconds:.6f}\n")
    return out.getvalue()
