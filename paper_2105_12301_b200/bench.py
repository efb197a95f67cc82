"""Kernel micro-benchmarks: (E, phase, seconds) rows over a dimension sweep.

Contract of the reference harness (pkg/src/crossmap/bench.py): ``run_bench``
takes the same arguments, enforces the same desk-scale bounds with the same
messages, draws the same seeded data and returns ``BenchRow(e, phase,
seconds)`` rows that ``bench_rows_to_csv`` renders as ``E,phase,seconds``.
What is timed is this package's device-backed API, so the paper's kernel
sweeps can be regenerated on a B200:

* ``knn`` -- per E the reference's two phases, "distance"
  (``pairwise_distances``, the materialised fp64 distance kernel) and "topk"
  (``partial_sort_topk``, CTA bitonic selection); ``fused=True`` adds "fused",
  the production ``build_knn_table`` sweep that never materialises the matrix.
* ``lookup`` -- per E one table of the library, then ``lookup_batch`` of all
  targets ("lookup").

Every call is synchronous, so a phase time includes the public API's
host<->device copies, as the reference's include its whole functions.
"""

from __future__ import annotations

from dataclasses import dataclass
from time import perf_counter
from typing import Callable, Iterator

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


def _check(kind: str, length: int, count: int, e_range, allow_large: bool) -> tuple[int, int]:
    if kind not in KINDS:
        raise ParameterError(f"unknown bench kind {kind!r}; choose from {KINDS}")
    lo, hi = (int(v) for v in e_range)
    if not 1 <= lo <= hi:
        raise ParameterError(f"bad dimension range {e_range}")
    if allow_large:
        return lo, hi
    limits = [("length", length, DESK_MAX_LENGTH)]
    if kind == "lookup":
        limits.append(("target count", count, DESK_MAX_SERIES))
    for what, value, bound in limits:
        if value > bound:
            raise ParameterError(f"{what} {value} exceeds the desk-scale bound {bound}; "
                                 f"pass allow_large to override")
    return lo, hi


def _knn_phases(library, spec, fused) -> Iterator[tuple[str, Callable[[], object]]]:
    """The knn phases of one dimension, in row order; "topk" consumes the matrix
    the "distance" phase produced."""
    state = {}
    yield "distance", lambda: state.__setitem__("d", pairwise_distances(library, spec))
    yield "topk", lambda: partial_sort_topk(state.pop("d"), spec.E + 1)
    if fused:
        yield "fused", lambda: build_knn_table(library, spec)


def _lookup_phases(library, targets, spec) -> Iterator[tuple[str, Callable[[], object]]]:
    table = build_knn_table(library, spec)  # untimed: the reference times the lookup alone
    yield "lookup", lambda: lookup_batch(table, targets)


def run_bench(kind: str, length: int = 4000, count: int = 1000,
              e_range: tuple[int, int] = (1, DEFAULT_E_MAX), seed: int = 0,
              workers: int | None = None, allow_large: bool = False,
              fused: bool = False) -> list[BenchRow]:
    """Time one kernel family across an embedding-dimension sweep.

    ``workers`` is accepted for signature compatibility: the GPU grid takes the
    place of the reference's thread pool."""
    lo, hi = _check(kind, length, count, e_range, allow_large)
    rng = np.random.default_rng(seed)
    library = rng.random(length)
    targets = list(rng.random((count, length))) if kind == "lookup" else None
    rows: list[BenchRow] = []
    for e in range(lo, hi + 1):
        spec = EmbeddingSpec(e, 1, e_max=max(hi, DEFAULT_E_MAX))
        phases = (_knn_phases(library, spec, fused) if kind == "knn"
                  else _lookup_phases(library, targets, spec))
        for phase, work in phases:
            t0 = perf_counter()
            work()
            rows.append(BenchRow(e, phase, perf_counter() - t0))
    return rows


def bench_rows_to_csv(rows: list[BenchRow]) -> str:
    """``E,phase,seconds`` text, six decimals (the reference's format)."""
    return "".join(["E,phase,seconds\n"] + [f"{r.e},{r.phase},{r.seconds:.6f}\n" for r in rows])
