"""Seeded synthetic series: the reference's generators, vectorised over series.

Input generation only (not on the hot path).  Every generator draws from
``np.random.default_rng(seed)`` (PCG64) exactly as pkg/src/crossmap/
synthetic.py:30-99 does, and the map iterations use the same float64
operation order, so single-series outputs are bit-identical to the
reference's (pinned in tests/test_synthetic.py against reference fixtures).
``mixed_dataset`` tiles the reference test suite's 20-series mix
(pkg/tests/conftest.py:7-23) to any N, which is how the benchmark shapes of
BASELINE.json are built.
"""

from __future__ import annotations

import numpy as np

from .embedding import Dataset, TimeSeries
from .errors import ParameterError, SeriesTooShortError

LOGISTIC_RATES = (3.58, 3.62, 3.7, 3.74, 3.82, 3.87, 3.92, 3.99)
COUPLINGS = (0.25, 0.35, 0.5)
SINE_PERIODS = (47.0, 131.0)
BLOCK = 20  # series per tile of the mix
BLOCK_SEED_STRIDE = 1000
DIVERGE_STRIDE = 1_000_003


def _length(n) -> int:
    if n < 1:
        raise SeriesTooShortError(f"length must be >= 1, got {n}")
    return int(n)


def uniform_noise(length: int, seed: int, low: float = 0.0, high: float = 1.0,
                  name: str = "noise") -> TimeSeries:
    _length(length)
    if not low < high:
        raise ParameterError(f"need low < high, got [{low}, {high})")
    return TimeSeries(np.random.default_rng(seed).uniform(low, high, size=length), name)


def _logistic_iter(v0: np.ndarray, r: np.ndarray, length: int) -> np.ndarray:
    out = np.empty((v0.size, length))
    v = v0.astype(np.float64).copy()
    for t in range(length):
        out[:, t] = v
        v = r * v * (1.0 - v)
    return out


def logistic_map(length: int, seed: int | None = None, r: float = 3.8, v0: float | None = None,
                 name: str = "logistic") -> TimeSeries:
    _length(length)
    if not 0.0 < r <= 4.0:
        raise ParameterError(f"logistic rate must lie in (0, 4], got {r}")
    if v0 is None:
        v0 = float(np.random.default_rng(seed).uniform(0.05, 0.95))
    if not 0.0 <= v0 <= 1.0:
        raise ParameterError(f"initial value must lie in [0, 1], got {v0}")
    return TimeSeries(_logistic_iter(np.array([v0]), np.array([float(r)]), length)[0], name)


def _coupled_iter(d0, y0, beta, length, r_d=3.8, r_y=3.5, burn_in=200, strict=True):
    d = np.asarray(d0, dtype=np.float64).copy()
    y = np.asarray(y0, dtype=np.float64).copy()
    beta = np.asarray(beta, dtype=np.float64)
    drv = np.empty((d.size, length))
    rsp = np.empty((d.size, length))
    with np.errstate(over="ignore", invalid="ignore"):
        for t in range(-burn_in, length):
            if t >= 0:
                drv[:, t] = d
                rsp[:, t] = y
            d, y = r_d * d * (1.0 - d), y * (r_y - r_y * y - beta * d)
    ok = np.all(np.isfinite(drv), axis=1) & np.all(np.isfinite(rsp), axis=1) & np.isfinite(y)
    if strict and not ok.all():
        raise ParameterError("coupled map diverged")
    return drv, rsp, ok


def coupled_logistic(length: int, seed: int, beta: float = 0.4, r_driver: float = 3.8,
                     r_response: float = 3.5, burn_in: int = 200) -> Dataset:
    _length(length)
    if not 0.0 <= beta <= 1.0:
        raise ParameterError(f"coupling strength must lie in [0, 1], got {beta}")
    rng = np.random.default_rng(seed)
    d0 = rng.uniform(0.1, 0.9)
    y0 = rng.uniform(0.1, 0.9)
    drv, rsp, _ = _coupled_iter([d0], [y0], [beta], length, r_driver, r_response, burn_in)
    return Dataset((TimeSeries(drv[0], "driver"), TimeSeries(rsp[0], "response")))


def mixed_dataset(n_series: int, length: int, seed: int = 2105, dtype=np.float32) -> np.ndarray:
    """(n_series, length) samples tiling the reference's 20-series mix.

    Block b (series 20b .. 20b+19) is pkg/tests/conftest.py's
    ``make_mixed_dataset(length, seed + 1000 b)``: 8 logistic maps
    (r = 3.58 .. 3.99), 3 coupled driver/response pairs (beta 0.25, 0.35, 0.5),
    4 uniform noises, 2 noisy sines (periods 47, 131).  Values are generated
    in float64 and rounded to ``dtype``.
    """
    if n_series < 1:
        raise ParameterError("need at least one series")
    L = _length(length)
    nb = (n_series + BLOCK - 1) // BLOCK
    seeds = seed + BLOCK_SEED_STRIDE * np.arange(nb)
    out = np.empty((nb * BLOCK, L), dtype=dtype)
    rows = np.arange(nb) * BLOCK
    # logistic maps, all blocks at once
    v0 = np.array([[np.random.default_rng(int(s) + p).uniform(0.05, 0.95) for p in range(8)] for s in seeds])
    r = np.broadcast_to(np.array(LOGISTIC_RATES), v0.shape)
    lg = _logistic_iter(v0.ravel(), r.ravel(), L).reshape(nb, 8, L)
    for p in range(8):
        out[rows + p] = lg[:, p]
    del lg
    # coupled pairs
    init = np.array([[np.random.default_rng(int(s) + 50 + q).uniform(0.1, 0.9, size=2) for q in range(3)]
                     for s in seeds])  # (nb, 3, 2)
    beta = np.broadcast_to(np.array(COUPLINGS), (nb, 3))
    drv, rsp, ok = _coupled_iter(init[..., 0].ravel(), init[..., 1].ravel(), beta.ravel(), L,
                                 strict=False)
    # A seed whose pair diverges (the reference raises, synthetic.py:92-97) is
    # replaced by seed + DIVERGE_STRIDE * attempt until the pair stays finite.
    for flat in np.flatnonzero(~ok):
        b, q = divmod(int(flat), 3)
        for attempt in range(1, 100):
            rng = np.random.default_rng(int(seeds[b]) + 50 + q + DIVERGE_STRIDE * attempt)
            d0, y0 = rng.uniform(0.1, 0.9), rng.uniform(0.1, 0.9)
            dd, rr, good = _coupled_iter([d0], [y0], [COUPLINGS[q]], L, strict=False)
            if good[0]:
                drv[flat], rsp[flat] = dd[0], rr[0]
                break
    drv = drv.reshape(nb, 3, L)
    rsp = rsp.reshape(nb, 3, L)
    for q in range(3):
        out[rows + 8 + 2 * q] = drv[:, q]
        out[rows + 9 + 2 * q] = rsp[:, q]
    del drv, rsp
    # noise
    for b, s in enumerate(seeds):
        for q in range(4):
            out[rows[b] + 14 + q] = np.random.default_rng(int(s) + 90 + q).uniform(0.0, 1.0, size=L)
    # noisy sines (one stream per block, drawn sine0 then sine1)
    steps = np.arange(L)
    base = [np.sin(2 * np.pi * steps / P) for P in SINE_PERIODS]
    for b, s in enumerate(seeds):
        rng = np.random.default_rng(int(s))
        for q in range(2):
            out[rows[b] + 18 + q] = base[q] + 0.05 * rng.standard_normal(L)
    return out[:n_series]


def gen_synthetic(kind: str, length: int, seed: int, params: dict | None = None) -> Dataset:
    params = dict(params or {})
    if kind == "uniform-noise":
        return Dataset((uniform_noise(length, seed, **params),))
    if kind == "logistic-map":
        return Dataset((logistic_map(length, seed, **params),))
    if kind == "coupled-logistic":
        return coupled_logistic(length, seed, **params)
    raise ParameterError(f"unknown synthetic kind {kind!r}")
