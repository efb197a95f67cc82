"""B200-native convergent cross mapping (kEDM's hot path, arXiv 2105.12301).

Drop-in for the reference package ``crossmap`` on its hot path: the same
classes and functions (re-exported below under the reference's names) plus
the kEDM-style entry points ``edim``, ``simplex``, ``xmap`` and ``ccm`` with
E / tau / Tp arguments.  All numerical work runs in hand-written sm_100a
kernels in ``libcmb200.so`` (see include/cmb200.h); there is no CPU fallback.
"""

from __future__ import annotations

__version__ = "0.1.0"

import numpy as np

from .embedding import (DEFAULT_E_MAX, Dataset, EmbeddingSpec, TimeSeries, as_values,
                        embedded_point, valid_count)
from .errors import (CrossmapError, CsvFormatError, DeviceError, ParameterError,
                     SeriesTooShortError, ZeroVarianceError)
from .pairwise import (LAYOUT_LIB_MAJOR, LAYOUT_TGT_MAJOR, CcmConfig, CcmStats, SkillMatrix,
                       ccm_pairwise, group_by_optimal_e, xmap)
from .skill import (OptimalEmbedding, PearsonAggregate, PredictionOutput, lookup_batch,
                    near_ties, optimal_embedding, pearson_stream, simplex_self_predict, skill_curves)
from .synthetic import coupled_logistic, gen_synthetic, logistic_map, mixed_dataset, uniform_noise
from .tables import (DistanceMatrix, NeighborTable, build_knn_table, normalize_to_weights,
                     oracle_knn, pairwise_distances, partial_sort_topk)
from . import binding  # noqa: E402  (needs __version__)
from .binding import CcmMatrix, EmbeddingSearch, ccm_matrix


def simplex(series, E: int, tau: int = 1, Tp: int = 1) -> float:
    """kEDM ``simplex``: self-prediction skill at dimension E, horizon Tp."""
    return binding.simplex(series, E, tau=tau, Tp=Tp)


def edim(values, E_max: int = DEFAULT_E_MAX, tau: int = 1, Tp: int = 1):
    """kEDM ``edim``: optimal embedding dimension by simplex self-prediction.

    1-D input -> ``EmbeddingSearch(e_star, skill_by_dim)`` (binding layout).
    2-D (time, series) input -> ``(e_star int32[N], rho float64[N, E_max])``
    computed in one batched device sweep; e_star 0 / NaN rho mark series whose
    skill is undefined (constant series).  ``near_ties(rho, e_star)`` lists the
    series whose best and runner-up skills differ by less than 1e-4.
    """
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim == 1:
        return binding.optimal_embedding(arr, E_max=E_max, tau=tau, Tp=Tp)
    if arr.ndim != 2:
        raise ParameterError(f"expected 1-D or 2-D (time, series) input, got shape {arr.shape}")
    if E_max < 1 or Tp < 1 or tau < 1:
        raise ParameterError(f"bad arguments E_max={E_max}, tau={tau}, Tp={Tp}")
    rho, est = skill_curves(np.ascontiguousarray(arr.T), E_max, tau, Tp)
    return est, rho


from . import convergence  # noqa: E402
from .convergence import Convergence, ccm, ccm_sweep  # noqa: E402  (kEDM ``ccm``)
from .io import (load_csv, read_skill_matrix, read_skill_matrix_npz,  # noqa: E402
                 write_skill_matrix, write_skill_matrix_device, write_skill_matrix_npz)
from .bench import BenchRow, run_bench  # noqa: E402  (kernel micro-benchmarks, bench.py)


__all__ = [
    "CcmConfig", "CcmMatrix", "CcmStats", "Convergence", "CrossmapError", "CsvFormatError", "DEFAULT_E_MAX",
    "Dataset", "DeviceError", "DistanceMatrix", "EmbeddingSearch", "EmbeddingSpec",
    "LAYOUT_LIB_MAJOR", "LAYOUT_TGT_MAJOR", "NeighborTable", "OptimalEmbedding", "ParameterError",
    "PearsonAggregate", "PredictionOutput", "SeriesTooShortError", "SkillMatrix", "TimeSeries",
    "ZeroVarianceError", "as_values", "build_knn_table", "ccm", "ccm_matrix", "ccm_pairwise", "ccm_sweep",
    "coupled_logistic", "edim", "embedded_point", "gen_synthetic", "group_by_optimal_e",
    "logistic_map", "lookup_batch", "mixed_dataset", "normalize_to_weights", "optimal_embedding",
    "near_ties", "oracle_knn", "pairwise_distances", "partial_sort_topk", "pearson_stream", "simplex",
    "simplex_self_predict", "skill_curves", "uniform_noise", "valid_count", "xmap",
    "load_csv", "read_skill_matrix", "read_skill_matrix_npz", "write_skill_matrix",
    "write_skill_matrix_device", "write_skill_matrix_npz", "BenchRow", "run_bench",
]
